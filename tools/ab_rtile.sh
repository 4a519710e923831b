#!/bin/bash
# Row groups per tile (SELLKIT_RTILE_GROUPS) on C1, C2 w=1/8, C5 w=8.
mkdir -p gpurun_out
out=gpurun_out/${1:-rtile}_ab.jsonl
: > $out
for rep in 1 2; do
for g in "" 1 2 4 16; do
  tag="rtile=$g"
  export SELLKIT_RTILE_GROUPS=$g
  [ -z "$g" ] && unset SELLKIT_RTILE_GROUPS
  python tools/stencil_step.py --points 5 --n 1000 --sigma 1 --w 1 --flush --reps 50 | sed "s/}$/, \"knob\": \"$tag\"}/" >> $out
  python tools/stencil_step.py --n 256 --w 1 | sed "s/}$/, \"knob\": \"$tag\"}/" >> $out
  python tools/stencil_step.py --n 256 --w 8 | sed "s/}$/, \"knob\": \"$tag\"}/" >> $out
  python tools/stencil_step.py --n 400 --w 8 --reps 30 | sed "s/}$/, \"knob\": \"$tag\"}/" >> $out
done
done
cat $out
