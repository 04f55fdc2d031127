#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=paper_2305_00515_b200/lib/libsobel5_b200.so
cp $L /tmp/orig.so
for v in build/variants/lib*.so; do
  cp $v $L; echo "== $v"; python tools/params_bench.py 2>&1 | grep -v "^$"
done
cp /tmp/orig.so $L
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
