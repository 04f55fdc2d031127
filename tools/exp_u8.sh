#!/bin/bash
# u8-only epilogue: GPU parity + u8 band sweep + bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CONTRACT=u8 BANDS=16,32,64,128 python tools/sweep.py > gpurun_out/u8_bands.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/u8_bands.txt
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print(d['value'], d['roofline']['frac'])
for k,v in d['variants'].items(): print(k, round(v['us'],1), round(v['gpx_s'],1), round(v['frac'],3))"
