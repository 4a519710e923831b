# Round-2 profile pass: C5 sweep-order A/B and ncu captures of the C5 headline kernel and
# the C3 KPM kernels; reports are reduced to CSV on the box (gpurun_out is capped at 64 MiB).
O=gpurun_out/r2m; mkdir -p $O
for r in 1 2 3; do
  python tools/stencil_step.py --n 400 --w 8 --reps 50 | sed 's/}$/, "lib": "rows"}/' >> $O/c5order.jsonl
  SELLKIT_AUTO_ORDER_L2=60000000 python tools/stencil_step.py --n 400 --w 8 --reps 50 | sed 's/}$/, "lib": "slab60M"}/' >> $O/c5order.jsonl
  SELLKIT_AUTO_ORDER_L2=30000000 python tools/stencil_step.py --n 400 --w 8 --reps 50 | sed 's/}$/, "lib": "slab30M"}/' >> $O/c5order.jsonl
done
csv() { ncu -i $1.ncu-rep --page raw --csv > $1_raw.csv 2>/dev/null; ncu -i $1.ncu-rep --page details --csv > $1_details.csv 2>/dev/null; }
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:spmv_tma_rows -s 3 -c 1 -o $O/c5 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c5.log 2>&1 && csv $O/c5
python tools/c3_step.py --dt c64 --reps 1 --warm 3 > $O/plain_c3c64.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:spmv_tma_rows -s 3 -c 1 -o $O/c3c64 python tools/c3_step.py --dt c64 --reps 1 --warm 3 > $O/ncu_c3c64.log 2>&1 && csv $O/c3c64 && rm -f $O/c3c64.ncu-rep
python tools/c3_step.py --dt r64 --reps 1 --warm 3 > $O/plain_c3r64.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:spmv_tma_rows -s 3 -c 1 -o $O/c3r64 python tools/c3_step.py --dt r64 --reps 1 --warm 3 > $O/ncu_c3r64.log 2>&1 && csv $O/c3r64 && rm -f $O/c3r64.ncu-rep
SELLKIT_AUTO_ORDER_L2=60000000 python tools/stencil_step.py --n 400 --w 8 --reps 1 --warm 3 > $O/plain_slab.log 2>&1 && SELLKIT_AUTO_ORDER_L2=60000000 ncu --set full --clock-control none -k regex:spmv_tma_rows -s 3 -c 1 -o $O/c5slab python tools/stencil_step.py --n 400 --w 8 --reps 1 --warm 3 > $O/ncu_slab.log 2>&1 && csv $O/c5slab && rm -f $O/c5slab.ncu-rep
du -sh $O > $O/du.txt
echo done > $O/rc.txt
