# A/B on epilogue (non-plain) and plain cases; usage: bash tools/ab_epi.sh OUTDIR lib...
O=$1; shift; mkdir -p $O
for r in 1 2 3; do
for lib in "$@"; do
  tag=$(basename $(dirname $lib))
  run() { SELLKIT_B200_LIB=$lib python tools/stencil_step.py "$@" | sed "s/}$/, \"lib\": \"$tag\"}/" >> $O/ab.jsonl 2>>$O/ab.err; }
  run --n 400 --w 8 --reps 30
  run --n 400 --w 8 --flags axpby --reps 20
  run --n 256 --w 8 --flags axpby --reps 20
  run --n 256 --w 32 --flags axpby --reps 20
  run --n 400 --w 1 --flags axpby --reps 20
  run --points 5 --n 1000 --sigma 1 --w 1 --flush --reps 50
  SELLKIT_B200_LIB=$lib python tools/c3_step.py --dt r64 --flags axpby --order $tag >> $O/ab.jsonl 2>>$O/ab.err
  SELLKIT_B200_LIB=$lib python tools/c3_step.py --dt c64 --flags axpby --order $tag >> $O/ab.jsonl 2>>$O/ab.err
done
done
