#!/bin/bash
# u8-only kernel: persistent double-buffered CTAs (SOBEL5_U8_PERSIST=1) vs one band per CTA
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${TAG:-u8p}
T=gpurun_out/${TAG}_time.txt; : > $T
for np in 2 4; do SOBEL5_U8_PERSIST=1 SOBEL5_U8_NP=$np timeout 300 python -m pytest tests/test_gpu_u8_only.py tests/test_gpu_detect.py -x -q 2>&1 | tail -1 | tee -a $T; done
for wh in "7680 4320" "3840 2160" "1920 1080"; do
  set -- $wh
  for np in 2 4; do for pe in 0 1; do
    echo "== ${1}x${2}: NP=$np persist=$pe" | tee -a $T
    W=$1 H=$2 SOBEL5_U8_PERSIST=$pe SOBEL5_U8_NP=$np BANDS=${BANDS:-8,16} GRAPH=1 CONTRACT=u8 timeout 300 python tools/sweep.py 2>&1 | tee -a $T
  done; done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sobel5_u8" -s 6 -c 1 -o gpurun_out/${TAG} -f env SOBEL5_U8_PERSIST=1 SOBEL5_U8_NP=2 SOBEL5_U8_BAND=16 CONTRACT=u8 python tools/sweep.py > /dev/null 2>&1
