# Round-end style validation without the ncu capture (kernel sources unchanged since the last one).
O=${1:-gpurun_out/val}; mkdir -p $O
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.jsonl 2> $O/bench.err; echo "bench $?" >> $O/rc.txt
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref.jsonl 2> $O/ref.err; echo "ref $?" >> $O/rc.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke $?" >> $O/rc.txt
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests $?" >> $O/rc.txt
timeout 900 python tools/bench_suite.py c1 c2 c3 c4 > $O/suite.jsonl 2> $O/suite.err; echo "suite $?" >> $O/rc.txt
