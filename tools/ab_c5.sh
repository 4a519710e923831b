# C5 plain A/B (alternating libs, many reps); usage: bash tools/ab_c5.sh OUTDIR lib...
O=$1; shift; mkdir -p $O
for r in 1 2 3 4; do
for lib in "$@"; do
  tag=$(basename $(dirname $lib))
  SELLKIT_B200_LIB=$lib python tools/stencil_step.py --n 400 --w 8 --reps 100 | sed "s/}$/, \"lib\": \"$tag\"}/" >> $O/ab.jsonl 2>>$O/ab.err
  SELLKIT_B200_LIB=$lib python tools/stencil_step.py --n 256 --w 8 --reps 100 | sed "s/}$/, \"lib\": \"$tag\"}/" >> $O/ab.jsonl 2>>$O/ab.err
  SELLKIT_B200_LIB=$lib python tools/stencil_step.py --n 256 --w 32 --reps 50 | sed "s/}$/, \"lib\": \"$tag\"}/" >> $O/ab.jsonl 2>>$O/ab.err
  SELLKIT_B200_LIB=$lib python tools/stencil_step.py --points 5 --n 1000 --sigma 1 --w 1 --flush --reps 50 | sed "s/}$/, \"lib\": \"$tag\"}/" >> $O/ab.jsonl 2>>$O/ab.err
done
done
