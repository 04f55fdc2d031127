#!/bin/bash
# C4 (256 x 1080p, one batched launch) band sweep, TMA rows vs register ring
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for b in 0 4 6 8 10 12; do
  echo -n "tma band=$b: "; SOBEL5_BAND=$b timeout 600 python bench.py --workload 1080p-batch --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), 'us', round(d['value'],1), round(d['roofline']['frac'],3))"
done
for b in 8 16; do
  echo -n "ring band=$b: "; SOBEL5_TMA_LOAD=0 SOBEL5_BAND=$b timeout 600 python bench.py --workload 1080p-batch --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), 'us', round(d['value'],1), round(d['roofline']['frac'],3))"
done
