#!/bin/bash
# e2e after the one-pass AVX-512 wire decode: 8K C3 and C4 frames, 3 repetitions
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -m pytest tests/test_gpu_wire16.py tests/test_gpu_frames.py -m gpu -q -x 2>&1 | tail -1
for rep in 1 2 3; do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('8K e2e', round(e['value'],3), 'Gpx/s', round(e['ms_per_step'],2), 'ms; cpp', d.get('e2e_cpp_api') and d['e2e_cpp_api']['value'])"
  python bench.py --steps 6 --warmup 3 --workload 1080p-batch --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('C4 e2e', round(e['value'],3), 'Gpx/s')"
done
