#!/bin/bash
# u8 kernel: packed-integer (U) vs packed-FP32 (SOBEL5_U8F=1) arithmetic,
# parity then timing per CTA width and band
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export GRAPH=1 CONTRACT=u8
for f in 1 0; do
  export SOBEL5_U8F=$f
  echo "==== U8F $f"
  python -m pytest tests/test_gpu_u8_only.py tests/test_gpu_detect.py -m gpu -x -q 2>&1 | tail -2
  for wv in 1 2 4; do
    export SOBEL5_U8_WARPS=$wv
    for wh in "7680 4320" "3840 2160" "1920 1080" "15360 8640"; do set -- $wh; echo "-- warps $wv $1x$2"; W=$1 H=$2 BANDS=0,8,16,24,32 python tools/sweep.py; done
  done
done
