#!/bin/bash
# Steady-state DRAM traffic per launch: ncu with --cache-control none over 8
# back-to-back launches (after 5 warm-up ones) of tools/sweep.py for each
# contract at 8K; tools/traffic.py averages them into profiles/traffic.json.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for c in sr sr32 u8; do
  timeout 600 ncu --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg \
    -k regex:"sobel5_(packed|u8)" -s 5 -c 8 --csv --log-file gpurun_out/traffic_$c.csv \
    env CONTRACT=$c python tools/sweep.py > /dev/null 2>&1
done
for c in 3sr 3u8; do
  cc=${c#3}
  timeout 600 ncu --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg \
    -k regex:"sobel3" -s 5 -c 8 --csv --log-file gpurun_out/traffic_$c.csv \
    env SOBEL3=1 CONTRACT=$( [ $cc = sr ] && echo sr3 || echo u8 ) python tools/sweep.py > /dev/null 2>&1
done
ls -la gpurun_out/traffic_*.csv
