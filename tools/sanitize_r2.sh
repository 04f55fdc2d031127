#!/bin/bash
# compute-sanitizer over the round-2 code paths (kernel U at every CTA width,
# the int16 wire, the ParityViolation CAS, TMA tensor stores, the multi-GPU
# C ABI), plus the round-1 subset.  memcheck / racecheck / synccheck.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T1="tests/test_gpu_parity.py::test_random_sweep_vs_oracle tests/test_gpu_parity.py::test_tma_band_loads_any_band tests/test_gpu_detect.py::test_pad_tma_band_loads tests/test_gpu_sobel3.py::test_sobel3_launch"
T2="tests/test_gpu_u8_only.py tests/test_gpu_parity.py::test_parity_violation_pair_matches_reference tests/test_gpu_tma_store.py tests/test_gpu_mgpu.py tests/test_gpu_detect.py tests/test_gpu_sobel3.py"
T3="tests/test_gpu_wire16.py"
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 5 --target-processes all \
    python -m pytest -q -x -p no:cacheprovider $T1 $T2 -k "not 4096" 2>&1 | tail -3
  echo "rc=${PIPESTATUS[0]}"
  for wv in 1 2; do
    SOBEL5_U8_WARPS=$wv timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 5 \
      python -m pytest -q -x -p no:cacheprovider tests/test_gpu_u8_only.py 2>&1 | tail -2
    echo "u8 warps $wv rc=${PIPESTATUS[0]}"
  done
done
echo "== memcheck: int16 wire host path"
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 5 \
  python -m pytest -q -x -p no:cacheprovider $T3 -k "61-97 or 300-1031 or staging or custom or split" 2>&1 | tail -3
echo "rc=${PIPESTATUS[0]}"
