# Round-end style validation on one fresh box: an ncu capture of the headline kernel first (its
# DRAM bytes become bench.py's roofline.traffic for these kernel sources), then the bench
# (driver command) + reference arm + smoke + the GPU suite + the secondary suite.
O=${1:-gpurun_out/final}; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_tma_rows -s 3 -c 1 -o $O/c5 \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
ncu -i $O/c5.ncu-rep --page details --csv > $O/c5_details.csv 2>/dev/null; echo "ncu $?" >> $O/rc.txt
python tools/ncu_summary.py $O/c5.ncu-rep --csv $O/c5_ncu.csv --traffic-key n400_w8_C32_s256_g1 > $O/c5_summary.txt 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json; rm -f $O/c5.ncu-rep
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.jsonl 2> $O/bench.err; echo "bench $?" >> $O/rc.txt
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref.jsonl 2> $O/ref.err; echo "ref $?" >> $O/rc.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke $?" >> $O/rc.txt
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests $?" >> $O/rc.txt
timeout 900 python tools/bench_suite.py c1 c2 c3 c4 > $O/suite.jsonl 2> $O/suite.err; echo "suite $?" >> $O/rc.txt
