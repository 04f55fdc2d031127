#!/bin/bash
# u8 kernel: warps per CTA (SOBEL5_U8_WARPS) x band, parity then timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export GRAPH=1 CONTRACT=u8
for wv in 1 2 4; do
  export SOBEL5_U8_WARPS=$wv
  echo "== warps $wv"
  python -m pytest tests/test_gpu_u8_only.py tests/test_gpu_detect.py -m gpu -x -q 2>&1 | tail -1
  for wh in "7680 4320" "3840 2160" "1920 1080" "15360 8640"; do set -- $wh; echo "-- $1x$2"; W=$1 H=$2 BANDS=0,8,16,24,32 python tools/sweep.py; done
done
