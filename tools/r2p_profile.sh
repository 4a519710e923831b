# stream microbenchmark, C2 w=32 / w=16 ncu captures (CSV on the box), secondary suite at HEAD
O=gpurun_out/r2p; mkdir -p $O
./tools/micro/stream_bw > $O/stream.jsonl 2>&1
csv() { ncu -i $1.ncu-rep --page raw --csv > $1_raw.csv 2>/dev/null; ncu -i $1.ncu-rep --page details --csv > $1_details.csv 2>/dev/null; rm -f $1.ncu-rep; }
python tools/stencil_step.py --n 256 --w 32 --reps 1 --warm 3 > $O/plain32.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:spmv_tma_rows -s 3 -c 1 -o $O/c2w32 python tools/stencil_step.py --n 256 --w 32 --reps 1 --warm 3 > $O/ncu32.log 2>&1 && csv $O/c2w32
python tools/stencil_step.py --n 256 --w 16 --reps 1 --warm 3 > $O/plain16.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:spmv_tma_rows -s 3 -c 1 -o $O/c2w16 python tools/stencil_step.py --n 256 --w 16 --reps 1 --warm 3 > $O/ncu16.log 2>&1 && csv $O/c2w16
timeout 900 python tools/bench_suite.py c1 c2 c3 c4 > $O/suite.jsonl 2> $O/suite.err
echo done > $O/rc.txt
