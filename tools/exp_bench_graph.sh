#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python bench.py --no-cpu-baseline > gpurun_out/bench_graph.json 2> gpurun_out/bench_graph.err
python bench.py --no-cpu-baseline --no-e2e --no-graph > gpurun_out/bench_nograph.json 2>&1
for wl in 1080p-batch 32k-bands 4k; do python bench.py --no-cpu-baseline --no-e2e --workload $wl --steps 50 | python -c "import json,sys; d=json.load(sys.stdin); print('$wl', round(d['value'],1), round(d['ms_per_step']*1e3,1), d['roofline']['frac'], d['gpu_launches'], d['config']['timed_as'])"; done
python -m pytest -q -x tests/test_gpu_bench_contract.py 2>&1 | tail -1
python -c "
import json
for f in ('gpurun_out/bench_graph.json','gpurun_out/bench_nograph.json'):
    d=json.load(open(f)); print(f, round(d['value'],1), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3), d['gpu_launches'], d['config']['timed_as'])
    for k,v in d['variants'].items(): print('  ', k, round(v['us'],1), round(v['frac'],3))
"
