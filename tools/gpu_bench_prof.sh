#!/bin/bash
# bench + ncu full captures of the SR kernel and the u8 (issue-bound) kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
TAG=${TAG:-u8}
CONTRACT=${CONTRACT:-u8} BANDS=${BANDS:-0} timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"sobel" -s 6 -c 1 -o gpurun_out/prof_$TAG -f python tools/sweep.py > gpurun_out/prof_$TAG.log 2>&1
tail -3 gpurun_out/prof_$TAG.log
cat gpurun_out/bench.json
