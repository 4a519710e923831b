# A/B of the dots-kernel variants (libs built into abtmp/ with EXTRA_NVFLAGS); usage: bash tools/ab_dots.sh OUTDIR lib...
O=$1; shift; mkdir -p $O
for r in 1 2; do
for lib in "$@"; do
  tag=$(basename $(dirname $lib))
  for dt in c64 r64; do SELLKIT_B200_LIB=$lib python tools/c3_step.py --dt $dt --order $tag >> $O/ab.jsonl 2>>$O/ab.err; done
  for w in 1 4 8 16; do SELLKIT_B200_LIB=$lib python tools/stencil_step.py --n 400 --w $w --flags dots | sed "s/}$/, \"lib\": \"$tag\"}/" >> $O/ab.jsonl 2>>$O/ab.err; done
  SELLKIT_B200_LIB=$lib python tools/stencil_step.py --n 256 --w 32 --flags kpm | sed "s/}$/, \"lib\": \"$tag\"}/" >> $O/ab.jsonl 2>>$O/ab.err
done
done
