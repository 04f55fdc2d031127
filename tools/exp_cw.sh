#!/bin/bash
# SR kernel A CTA width (SOBEL5_CTA_WARPS builds) at 4K / 1080p: register ring and TMA rows x band
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export GRAPH=1
for v in default cw2 cw1; do
  if [ "$v" = default ]; then unset SOBEL5_LIB; else export SOBEL5_LIB=$PWD/build/variants/$v/libsobel5_b200.so; fi
  for wh in "3840 2160" "1920 1080"; do set -- $wh
    echo "== $v $1x$2 ring"; SOBEL5_TMA_LOAD=0 W=$1 H=$2 BANDS=4,8,12,16,24,32 python tools/sweep.py
    echo "== $v $1x$2 tma";  W=$1 H=$2 BANDS=4,6,8,12,16 python tools/sweep.py
  done
done
