#!/bin/bash
# end-of-round measurement package on one B200: bench line, reference arm,
# launch list of the bench command (ncu, per-launch durations only)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench_rc=$? >> gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo ref_rc=$? >> gpurun_out/final_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e > gpurun_out/final_ncu.log 2>&1; echo ncu_rc=$? >> gpurun_out/final_ncu.log
echo done
