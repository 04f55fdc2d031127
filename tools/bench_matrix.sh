#!/bin/bash
# every bench.py workload x contract x prefetch combination runs and prints one line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for wl in 8k 4k 1080p-batch 32k-bands; do for c in sr sr32 u8; do for pf in 1 0; do
  out=$(timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $wl --contract $c --prefetch $pf --steps 10 --warmup 3 2>&1 | tail -1)
  echo "$wl $c pf=$pf $(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3), d['gpu_launches'])" 2>&1 | tail -1)"
done; done; done
