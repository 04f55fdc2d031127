#!/bin/bash
# u8 kernel variants (tools/build_variant.sh): parity of the u8 tests, then 8K/4K/1080p timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export GRAPH=1 CONTRACT=u8
for v in default u8w2 u8gd u8gdw2; do
  if [ "$v" = default ]; then unset SOBEL5_LIB; else export SOBEL5_LIB=$PWD/build/variants/$v/libsobel5_b200.so; fi
  echo "== $v"
  python -m pytest tests/test_gpu_u8_only.py -m gpu -x -q 2>&1 | tail -1
  for wh in "7680 4320" "3840 2160" "1920 1080"; do set -- $wh; W=$1 H=$2 BANDS=0,16 python tools/sweep.py; done
done
