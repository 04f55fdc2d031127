#!/bin/bash
# ncu --set full of one launch of the 8K kernel (env: CONTRACT, BANDS, PFS, TAG)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${TAG:-prof}
BANDS=${BANDS:-16} PFS=${PFS:-1} timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"sobel5_(packed|stream)" -s 6 -c 1 -o gpurun_out/$TAG -f python tools/sweep.py > gpurun_out/$TAG.log 2>&1
tail -2 gpurun_out/$TAG.log
