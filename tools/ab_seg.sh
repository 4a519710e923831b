# dynamic-deal segment size A/B (SELLKIT_TMA_SEG), burst regime; usage: bash tools/ab_seg.sh OUTDIR
O=$1; mkdir -p $O
for r in 1 2 3; do
for seg in 1 2 4 8; do
  run() { SELLKIT_TMA_SEG=$seg python tools/stencil_step.py "$@" --reps 20 | sed "s/}$/, \"lib\": \"seg$seg\"}/" >> $O/ab.jsonl 2>>$O/ab.err; }
  run --n 400 --w 8
  run --n 400 --w 8 --flags axpby
  run --n 256 --w 16
  run --n 256 --w 32
  run --n 256 --w 8 --flags axpby
  SELLKIT_TMA_SEG=$seg python tools/c3_step.py --dt r64 --flags axpby --order seg$seg >> $O/ab.jsonl 2>>$O/ab.err
  SELLKIT_TMA_SEG=$seg python tools/c3_step.py --dt c64 --flags axpby --order seg$seg >> $O/ab.jsonl 2>>$O/ab.err
done
done
