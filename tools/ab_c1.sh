#!/bin/bash
# C1 (5-pt 1000^2, SELL-32-1, w = 1, L2 flushed) under the kernel-choice knobs.
mkdir -p gpurun_out
out=gpurun_out/${1:-c1}_ab.jsonl
: > $out
for rep in 1 2; do
for cfg in "" "SELLKIT_SPMV_KERNEL=ldg" "SELLKIT_TMA_SEG=2" "SELLKIT_TMA_SEG=4"; do
  env $cfg python tools/bench_suite.py c1 | sed "s/^{/{\"knob\": \"$cfg\", /" >> $out
done
done
cat $out
