#!/bin/bash
# sobel5_run_host through the frame ring (default) vs the whole-image staging
# (SOBEL5_RUN_HOST_RING=0): parity of the host paths, then 8K / C4 e2e x3
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -m pytest tests/test_gpu_wire16.py tests/test_gpu_frames.py tests/test_gpu_parity.py tests/test_cpp_api.py tests/test_cpp_acceptance.py tests/test_gpu_bench_contract.py -m gpu -q -x 2>&1 | tail -1
for rep in 1 2 3; do
  for ring in 1 0; do
    SOBEL5_RUN_HOST_RING=$ring python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('ring $ring 8K e2e', round(e['value'],3), 'Gpx/s', round(e['ms_per_step'],2), 'ms d2h', e['d2h_bytes_per_step'])"
  done
  python bench.py --steps 6 --warmup 3 --workload 1080p-batch --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('C4 e2e', round(e['value'],3), 'Gpx/s')"
done
