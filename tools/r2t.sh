O=gpurun_out/r2t; mkdir -p $O
timeout 600 python -m pytest tests/test_sweep_order_gpu.py -q > $O/tests.log 2>&1
for r in 1 2; do
  for dt in c64 r64; do python tools/c3_step.py --dt $dt --order auto >> $O/ab.jsonl; done
  for cfg in "--n 400 --w 8" "--n 400 --w 16" "--n 320 --w 16" "--n 256 --w 32" "--n 256 --w 16" "--n 256 --w 8"; do
    python tools/stencil_step.py $cfg --reps 20 | sed "s/}$/, \"lib\": \"auto\"}/" >> $O/ab.jsonl
  done
done
