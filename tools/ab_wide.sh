#!/bin/bash
# RHS rows of 512 B / 1 KB: rows kernel with wide lane vectors (abtmp/wide) vs the column-slice kernel
# (abtmp/base: 2 CTAs/SM, abtmp/minb1: 1 CTA/SM); C3 TI matrix, complex and real, plain and KPM.
mkdir -p gpurun_out; out=gpurun_out/${1:-wide}_ab.jsonl; : > $out
for rep in 1 2; do
for lib in abtmp/base abtmp/minb1 abtmp/wide; do
  tag=$(basename $lib)
  for cfg in "c64 32" "c64 64" "r64 64"; do
    set -- $cfg
    for fl in plain kpm; do
      SELLKIT_B200_LIB=$lib/libsellkit_b200.so python tools/c3_step.py --dt $1 --w $2 --flags $fl --reps 10 --order $tag >> $out
    done
  done
done
done
