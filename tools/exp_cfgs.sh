#!/bin/bash
# bench lines for the BASELINE configs at N=1: C3 (default, with sizes C1/C2), C4 batch, C5 32K
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -m pytest tests/test_gpu_wire16.py tests/test_gpu_bench_contract.py -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/cfg_c3.json 2> gpurun_out/cfg_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --workload 1080p-batch --steps 20 --no-cpu-baseline > gpurun_out/cfg_c4.json 2> gpurun_out/cfg_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --workload 32k-bands --steps 10 --no-cpu-baseline > gpurun_out/cfg_c5.json 2> gpurun_out/cfg_c5.err; echo "c5 rc=$?"
