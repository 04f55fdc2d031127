#!/bin/bash
# Round-2 measurement package: bench line, ncu launch list of the bench
# command, ncu --set full of the headline SR kernel and of the u8 kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nproc > gpurun_out/r2_host.txt; lscpu | head -20 >> gpurun_out/r2_host.txt
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/r2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/r2_launches_bench.log 2>&1
echo "launch list rc=$?"
CONTRACT=sr BANDS=0 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"sobel5_packed" -s 6 -c 1 -o gpurun_out/r2_prof_sr -f python tools/sweep.py > gpurun_out/r2_prof_sr.log 2>&1
echo "sr prof rc=$?"
CONTRACT=u8 BANDS=0 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"sobel5_u8" -s 6 -c 1 -o gpurun_out/r2_prof_u8 -f python tools/sweep.py > gpurun_out/r2_prof_u8.log 2>&1
echo "u8 prof rc=$?"
