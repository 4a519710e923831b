# Checked build (device bounds assertions, SK_CHECK=1) into abtmp/check and the GPU suite
# against it -- the stand-in for compute-sanitizer memcheck (closed on this pool).
#   bash tools/check_build.sh build      (here: nvcc only)
#   bash tools/check_build.sh run OUTDIR (GPU box)
set -e
if [ "$1" = build ]; then
  make -j8 -C paper_1507_08101_b200/csrc OUTDIR=$(pwd)/abtmp/check OBJDIR=/tmp/obj_check \
       BIN=$(pwd)/abtmp/check/spmvbench EXTRA_NVFLAGS="-DSK_CHECK=1 -lineinfo"
  rm -rf /tmp/obj_check
else
  O=${2:-gpurun_out/check}; mkdir -p $O
  SELLKIT_B200_LIB=abtmp/check/libsellkit_b200.so timeout 2400 python -m pytest tests -m gpu -q \
      --deselect tests/test_fullsize_real_gpu.py > $O/check_tests.log 2>&1 || true
  tail -3 $O/check_tests.log
fi
