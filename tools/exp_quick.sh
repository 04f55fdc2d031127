#!/bin/bash
# quick timing: 8K SR / u8 (band default), params (1,1,1,1), + GPU parity of the packed kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for c in sr u8; do CONTRACT=$c python tools/sweep.py 2>&1 | tail -1; done
python tools/params_bench.py 2>&1 | grep "1, 1, 1, 1) generic=0"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_u8_only.py tests/test_gpu_detect.py -x -q 2>&1 | tail -2
