O=gpurun_out/r2ah; mkdir -p $O
csv() { ncu -i $1.ncu-rep --page raw --csv > $1_raw.csv 2>/dev/null; rm -f $1.ncu-rep; }
SELLKIT_B200_LIB=abtmp/dynplain/libsellkit_b200.so python tools/stencil_step.py --n 400 --w 8 --reps 1 --warm 3 > $O/p1.log 2>&1 && SELLKIT_B200_LIB=abtmp/dynplain/libsellkit_b200.so ncu --set full --clock-control none -k regex:spmv_tma_rows -s 3 -c 1 -o $O/dyn python tools/stencil_step.py --n 400 --w 8 --reps 1 --warm 3 > $O/n1.log 2>&1 && csv $O/dyn
python tools/stencil_step.py --n 400 --w 8 --reps 1 --warm 3 > $O/p2.log 2>&1 && ncu --set full --clock-control none -k regex:spmv_tma_rows -s 3 -c 1 -o $O/static python tools/stencil_step.py --n 400 --w 8 --reps 1 --warm 3 > $O/n2.log 2>&1 && csv $O/static
