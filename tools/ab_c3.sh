# A/B of library variants on the C3 KPM step and the stencil dots cases; usage: bash tools/ab_c3.sh OUTDIR lib...
O=$1; shift; mkdir -p $O
for r in 1 2; do
for lib in "$@"; do
  tag=$(basename $(dirname $lib))
  for dt in c64 r64; do SELLKIT_B200_LIB=$lib python tools/c3_step.py --dt $dt --order $tag >> $O/ab.jsonl 2>>$O/ab.err; done
  for w in 8 16; do SELLKIT_B200_LIB=$lib python tools/stencil_step.py --n 400 --w $w --flags dots | sed "s/}$/, \"lib\": \"$tag\"}/" >> $O/ab.jsonl 2>>$O/ab.err; done
done
done
