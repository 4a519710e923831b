#!/bin/bash
# Lane vector width of the rows kernel (SK_RVEC 32 vs 64 B, the latter at 4 or 3 CTAs/SM).
mkdir -p gpurun_out; out=gpurun_out/${1:-rvec}_ab.jsonl; : > $out
for rep in 1 2; do
for lib in abtmp/base abtmp/rv64 abtmp/rv64m3; do
  tag=$(basename $lib)
  run() { SELLKIT_B200_LIB=$lib/libsellkit_b200.so python tools/stencil_step.py "$@" | sed "s/}$/, \"lib\": \"$tag\"}/" >> $out; }
  for w in 8 16 32; do run --n 256 --w $w; done
  run --n 400 --w 8 --reps 30
  run --n 256 --w 16 --flags axpby
  SELLKIT_B200_LIB=$lib/libsellkit_b200.so python tools/c3_step.py --dt c64 --flags plain --order $tag >> $out
  SELLKIT_B200_LIB=$lib/libsellkit_b200.so python tools/c3_step.py --dt c64 --order $tag >> $out
done
done
