#!/bin/bash
# Small-image SR efficiency: PDL on/off x band x TMA rows, CUDA-graph timing (tools/sweep.py GRAPH=1)
cd "$(dirname "$0")/.."
export GRAPH=1
for pdl in 0 1; do
  for wh in "3840 2160" "1920 1080" "7680 4320"; do
    set -- $wh
    echo "== ${1}x${2} SR PDL=$pdl default"
    SOBEL5_PDL=$pdl W=$1 H=$2 BANDS=0 python tools/sweep.py
    echo "== ${1}x${2} SR PDL=$pdl TMA rows, bands 4,6,8,12,16"
    SOBEL5_PDL=$pdl W=$1 H=$2 BANDS=4,6,8,12,16 python tools/sweep.py
    echo "== ${1}x${2} SR PDL=$pdl register ring, bands 4,8,12,16,24,32"
    SOBEL5_TMA_LOAD=0 SOBEL5_PDL=$pdl W=$1 H=$2 BANDS=4,8,12,16,24,32 python tools/sweep.py
    echo "== ${1}x${2} u8 PDL=$pdl default"
    CONTRACT=u8 SOBEL5_PDL=$pdl W=$1 H=$2 BANDS=0 python tools/sweep.py
  done
done
