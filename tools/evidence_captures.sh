# ncu --set full captures of the secondary configurations' dominant kernels (CSV kept, reports
# deleted): C3 C64 / R64 KPM step and C2 w = 16 / 32 plain.  Usage: bash tools/evidence_captures.sh OUTDIR
O=${1:-gpurun_out/ev}; mkdir -p $O
cap() {  # name, command...
  local n=$1; shift
  "$@" > $O/${n}_plain.log 2>&1 && \
  ncu --set full --clock-control none -k regex:spmv_tma_rows -s 3 -c 1 -o $O/$n "$@" > $O/${n}_ncu.log 2>&1
  ncu -i $O/$n.ncu-rep --page details --csv > $O/${n}_details.csv 2>/dev/null
  python tools/ncu_summary.py $O/$n.ncu-rep > $O/${n}_summary.jsonl 2>/dev/null
  rm -f $O/$n.ncu-rep
}
cap c3c64 python tools/c3_step.py --dt c64 --reps 3 --warm 3
cap c3r64 python tools/c3_step.py --dt r64 --reps 3 --warm 3
cap c2w32 python tools/stencil_step.py --n 256 --w 32 --reps 3 --warm 3
cap c2w16 python tools/stencil_step.py --n 256 --w 16 --reps 3 --warm 3
