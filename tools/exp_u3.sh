#!/bin/bash
# 3x3 u8-only kernel (sobel3_u8.cuh): parity, then warps x band timing vs kernel C
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -m pytest tests/test_gpu_u8_only.py tests/test_gpu_sobel3.py tests/test_gpu_detect.py -m gpu -x -q 2>&1 | tail -1
export GRAPH=1 CONTRACT=u8 SOBEL3=1
for wh in "7680 4320" "3840 2160" "1920 1080" "15360 8640"; do
  set -- $wh
  echo "-- $1x$2 kernel C (SOBEL5_U8_FAST=0)"; SOBEL5_U8_FAST=0 W=$1 H=$2 BANDS=0 python tools/sweep.py
  for wv in 1 2 4; do echo "-- $1x$2 U3 warps $wv"; SOBEL5_U8_WARPS=$wv W=$1 H=$2 BANDS=0,8,16,24,32 python tools/sweep.py; done
done
