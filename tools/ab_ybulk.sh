#!/bin/bash
# y through shared memory + bulk stores (SK_YBULK=1 build) vs STG, plain sweeps of the wide plans.
mkdir -p gpurun_out; out=gpurun_out/${1:-ybulk}_ab.jsonl; : > $out
for rep in 1 2; do
for lib in abtmp/base abtmp/ybulk; do
  tag=$(basename $lib)
  for w in 8 16 32; do SELLKIT_B200_LIB=$lib/libsellkit_b200.so python tools/stencil_step.py --n 256 --w $w | sed "s/}$/, \"lib\": \"$tag\"}/" >> $out; done
  SELLKIT_B200_LIB=$lib/libsellkit_b200.so python tools/stencil_step.py --n 400 --w 8 --reps 30 | sed "s/}$/, \"lib\": \"$tag\"}/" >> $out
  SELLKIT_B200_LIB=$lib/libsellkit_b200.so python tools/c3_step.py --dt c64 --flags plain --order $tag >> $out
  SELLKIT_B200_LIB=$lib/libsellkit_b200.so python tools/c3_step.py --dt r64 --flags plain --order $tag >> $out
done
done
