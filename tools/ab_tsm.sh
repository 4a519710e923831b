# A/B of TSM variants on the C4 shapes (N = 1e8); usage: bash tools/ab_tsm.sh OUTDIR "m list" lib...
O=$1; shift; MS=$1; shift; mkdir -p $O
for r in 1 2; do
for lib in "$@"; do
  tag=$(basename $(dirname $lib))
  SELLKIT_B200_LIB=$lib python tools/tsm_case.py $MS | sed "s/}$/, \"lib\": \"$tag\"}/" >> $O/ab.jsonl 2>>$O/ab.err
done
done
