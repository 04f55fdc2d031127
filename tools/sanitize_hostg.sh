#!/bin/bash
# compute-sanitizer over the late round-2 host paths: the int16 wire without g
# (kernels 15|kOutN16 and the 3x3 gx|gy|kOutN16), g rebuilt on the host, the
# frames engine.  memcheck / racecheck / synccheck.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T="tests/test_gpu_wire16.py tests/test_gpu_frames.py"
K="61-97 or 300-1031 or 300-517 or 5-5 or custom or split or staging or planes or errors or 2100-2060"
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 5 --target-processes all \
    python -m pytest -q -x -p no:cacheprovider $T -k "$K" 2>&1 | tail -2
  echo "rc=${PIPESTATUS[0]}"
done
