# A/B in the burst regime (20 reps after 3 warm-ups, like the driver's bench), alternating libs
# usage: bash tools/ab_burst.sh OUTDIR lib...
O=$1; shift; mkdir -p $O
for r in 1 2 3 4; do
for lib in "$@"; do
  tag=$(basename $(dirname $lib))
  run() { SELLKIT_B200_LIB=$lib python tools/stencil_step.py "$@" --reps 20 | sed "s/}$/, \"lib\": \"$tag\"}/" >> $O/ab.jsonl 2>>$O/ab.err; }
  run --n 400 --w 8
  run --n 400 --w 1
  run --n 320 --w 8
  for w in 1 4 8 16 32; do run --n 256 --w $w; done
  run --points 5 --n 1000 --sigma 1 --w 1 --flush
done
done
