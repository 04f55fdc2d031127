#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for round in 1 2 3; do for t in 0 1; do for c in sr u8; do
  echo "$round tma=$t $c $(SOBEL5_TMA_LOAD=$t CONTRACT=$c python tools/sweep.py | tail -1)"
done; done; done
SOBEL5_TMA_LOAD=1 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_u8_only.py tests/test_gpu_host_paths.py 2>&1 | tail -2
