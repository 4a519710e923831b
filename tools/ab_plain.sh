# A/B of library variants on the plain SpMMV cases (C1, C2 widths, C5); usage: bash tools/ab_plain.sh OUTDIR lib...
O=$1; shift; mkdir -p $O
for r in 1 2; do
for lib in "$@"; do
  tag=$(basename $(dirname $lib))
  run() { SELLKIT_B200_LIB=$lib python tools/stencil_step.py "$@" | sed "s/}$/, \"lib\": \"$tag\"}/" >> $O/ab.jsonl 2>>$O/ab.err; }
  for w in 1 4 8 16 32; do run --n 256 --w $w; done
  run --n 400 --w 8 --reps 50
  run --points 5 --n 1000 --sigma 1 --w 1 --flush --reps 50
done
done
