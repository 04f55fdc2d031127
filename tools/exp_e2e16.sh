#!/bin/bash
# e2e with the host pool on every core: g rebuilt vs shipped, row chunks per 8K frame
cd "${GRAFT_REPO_ROOT:-/root/repo}"
e2e() { python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(round(e['value'],3), 'Gpx/s', round(e.get('ms_per_step', 0),2), 'ms', 'cpp', d.get('e2e_cpp_api', {}).get('value'))"; }
for rep in 1 2; do
for g in 1 0; do
  for c in 8 16 32; do
    echo "WIRE_G=$g CHUNKS=$c $(SOBEL5_WIRE_G=$g SOBEL5_CHUNKS=$c e2e)"
  done
  echo "WIRE_G=$g C4 $(SOBEL5_WIRE_G=$g e2e --workload 1080p-batch --steps 6 --warmup 3)"
done
done
