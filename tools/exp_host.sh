#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_host_paths.py tests/test_gpu_parity.py tests/test_cpp_api.py -x -q -m gpu > gpurun_out/pytest_host.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_host.log
tail -5 gpurun_out/pytest_host.log
./build/cpp_e2e 7680 4320 10 | tee gpurun_out/cpp_e2e.json
./build/cpp_e2e 3840 2160 10
./build/cpp_e2e 1920 1080 20
