#!/bin/bash
# Column-slice kernel for >= 512-B RHS rows at 2 vs 1 CTA/SM (SK_MINB_WIDE): complex double w = 32 / 64.
mkdir -p gpurun_out; out=gpurun_out/${1:-minb}_ab.jsonl; : > $out
for rep in 1 2; do
for lib in abtmp/base abtmp/minb1; do
  tag=$(basename $lib)
  for w in 32 64; do
    for fl in plain kpm; do
      SELLKIT_B200_LIB=$lib/libsellkit_b200.so python tools/c3_step.py --dt c64 --w $w --flags $fl --reps 10 --order $tag >> $out
    done
  done
  SELLKIT_B200_LIB=$lib/libsellkit_b200.so python tools/c3_step.py --dt r64 --w 64 --flags plain --reps 10 --order $tag >> $out
done
done
