#!/bin/bash
# host pool size (SOBEL5_HOST_THREADS) x e2e: 8K C3 (sobel5_run_host) and C4 frames
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2; do
for t in 8 12 16; do
  export SOBEL5_HOST_THREADS=$t
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('threads $t 8K e2e', round(d['e2e']['value'],3), round(d['e2e']['ms_per_step'],2), 'ms')"
  python bench.py --steps 6 --warmup 3 --workload 1080p-batch --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('threads $t C4 e2e', round(d['e2e']['value'],3))"
done
done
