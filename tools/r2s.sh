O=gpurun_out/r2s; mkdir -p $O
for r in 1 2; do
for l2 in 126000000 60000000 30000000 15000000; do
  for dt in c64 r64; do SELLKIT_AUTO_ORDER_L2=$l2 python tools/c3_step.py --dt $dt --order slab$l2 >> $O/ab.jsonl; done
  for cfg in "--n 400 --w 16" "--n 320 --w 16" "--n 256 --w 32" "--n 256 --w 16"; do
    SELLKIT_AUTO_ORDER_L2=$l2 python tools/stencil_step.py $cfg --reps 20 | sed "s/}$/, \"lib\": \"slab$l2\"}/" >> $O/ab.jsonl
  done
done
done
