#!/bin/bash
# Lanes per 512-B / 1-KB RHS row (SK_WIDE_LANES 8 / 16 / 32 builds in abtmp/l8, l16, l32).
mkdir -p gpurun_out; out=gpurun_out/${1:-lanes}_ab.jsonl; : > $out
for rep in 1 2; do
for lib in ${LIBS:-abtmp/l8 abtmp/l16 abtmp/l32}; do
  tag=$(basename $lib)
  for cfg in "c64 32" "c64 64" "r64 64"; do
    set -- $cfg
    for fl in plain axpby kpm; do
      SELLKIT_B200_LIB=$lib/libsellkit_b200.so python tools/c3_step.py --dt $1 --w $2 --flags $fl --reps 10 --order $tag >> $out
    done
  done
done
done
