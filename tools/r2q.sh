O=gpurun_out/r2q; mkdir -p $O
for r in 1 2; do
for w in 32 16; do
  python tools/stencil_step.py --n 256 --w $w --reps 30 | sed 's/}$/, "lib": "rows"}/' >> $O/ab.jsonl
  for l2 in 80000000 60000000 40000000; do
    SELLKIT_AUTO_ORDER_L2=$l2 python tools/stencil_step.py --n 256 --w $w --reps 30 | sed "s/}$/, \"lib\": \"slab$l2\"}/" >> $O/ab.jsonl
  done
done
done
