#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for c in u8; do
CONTRACT=$c BANDS=${BANDS:-32,40,48,56,64,72,80,89,96} python tools/sweep.py 2>&1
done
echo "== 3x3 u8"
SOBEL3=1 CONTRACT=u8 BANDS=${BANDS3:-32,48,64,89,96,128} python tools/sweep.py 2>&1
