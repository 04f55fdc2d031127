#!/bin/bash
# StreamResult through TMA tensor stores (SOBEL5_TS=1: per-CTA boxes,
# 2: per-warp boxes) vs register stores (SOBEL5_TS=0): parity tests,
# CUDA-graph timing, ncu of one TS launch.  SIZES="7680x4320 ...", TSB="bands".
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${TAG:-ts}
T=gpurun_out/${TAG}_time.txt; : > $T
for mode in ${TSMODES:-1 2}; do
  SOBEL5_TS=$mode timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_host_paths.py tests/test_gpu_stress.py -x -q 2>&1 | tail -1 | sed "s/^/TS=$mode /" | tee -a $T
done
for wh in ${SIZES:-7680x4320}; do
  W=${wh%x*}; H=${wh#*x}
  echo "== ${W}x${H}: register stores (TS=0, default band)" | tee -a $T
  W=$W H=$H SOBEL5_TS=0 GRAPH=1 CONTRACT=sr timeout 300 python tools/sweep.py 2>&1 | tee -a $T
  for mode in ${TSMODES:-1 2}; do
    echo "== ${W}x${H}: TMA tensor stores mode $mode" | tee -a $T
    for b in ${TSB:-2 4 6 8}; do
      W=$W H=$H SOBEL5_TS=$mode SOBEL5_TS_BAND=$b GRAPH=1 CONTRACT=sr timeout 300 python tools/sweep.py 2>&1 | sed "s/^/tsband=$b /" | tee -a $T
    done
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sobel5_packed" -s 6 -c 1 -o gpurun_out/${TAG} -f env SOBEL5_TS=${NCU_TS:-2} CONTRACT=sr python tools/sweep.py > /dev/null 2>&1
