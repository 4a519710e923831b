O=gpurun_out/r2r; mkdir -p $O
for r in 1 2; do
for cfg in "--n 400 --w 8" "--n 400 --w 16" "--n 256 --w 8" "--n 320 --w 8" "--n 320 --w 16"; do
  python tools/stencil_step.py $cfg --reps 20 | sed 's/}$/, "lib": "rows"}/' >> $O/ab.jsonl
  for l2 in 120000000 60000000 30000000 15000000; do
    SELLKIT_AUTO_ORDER_L2=$l2 python tools/stencil_step.py $cfg --reps 20 | sed "s/}$/, \"lib\": \"slab$l2\"}/" >> $O/ab.jsonl
  done
done
done
