#!/bin/bash
# u8-only kernels (sobel5_u8.cuh): parity, A/B timing (CUDA graph) of the
# general packed kernel (SOBEL5_U8_FAST=0), the band kernel (SOBEL5_U8_KERNEL=1)
# and the persistent stream kernel (default), one ncu --set full capture.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${TAG:-u8fast}
timeout 600 python -m pytest tests/test_gpu_u8_only.py tests/test_gpu_detect.py "tests/test_gpu_parity.py::test_epilogue_arithmetic_exhaustive" -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
T=gpurun_out/${TAG}_time.txt; : > $T
for wh in "7680 4320" "3840 2160" "1920 1080"; do
  set -- $wh
  echo "== ${1}x${2}: packed / band16 / stream(minrows ${MINROWS:-16 32 64})" | tee -a $T
  W=$1 H=$2 SOBEL5_U8_FAST=0 GRAPH=1 CONTRACT=u8 timeout 300 python tools/sweep.py 2>&1 | tee -a $T
  W=$1 H=$2 SOBEL5_U8_KERNEL=1 BANDS=16 GRAPH=1 CONTRACT=u8 timeout 300 python tools/sweep.py 2>&1 | tee -a $T
  for mr in ${MINROWS:-16 32 64}; do
    W=$1 H=$2 SOBEL5_U8_MINROWS=$mr GRAPH=1 CONTRACT=u8 timeout 300 python tools/sweep.py 2>&1 | tee -a $T
  done
done
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sobel5_u8" -s 6 -c 1 \
  -o gpurun_out/${TAG} -f env CONTRACT=u8 python tools/sweep.py > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
fi
