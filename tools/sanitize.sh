#!/bin/bash
# compute-sanitizer over representative GPU tests (memcheck: out-of-bounds /
# misaligned global+shared accesses incl. TMA; racecheck: shared memory;
# synccheck: barriers).  Small shapes only: the sanitizer is ~100x slower.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T="tests/test_gpu_parity.py::test_random_sweep_vs_oracle tests/test_gpu_parity.py::test_tma_band_loads_any_band tests/test_gpu_parity.py::test_plane_pitch_variants tests/test_gpu_detect.py::test_pad_tma_band_loads tests/test_gpu_u8_only.py::test_u8_only_valid tests/test_gpu_f32.py::test_f32_pad tests/test_gpu_sobel3.py::test_sobel3_launch tests/test_gpu_parity.py::test_row_band_partition_equals_whole"
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 5 --target-processes all \
    python -m pytest -q -x -p no:cacheprovider $T 2>&1 | tail -4
  echo "rc=${PIPESTATUS[0]}"
done
