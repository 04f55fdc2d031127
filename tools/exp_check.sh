#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -m pytest tests/test_gpu_u8_only.py tests/test_gpu_detect.py tests/test_gpu_baseline_sizes.py -m gpu -x -q 2>&1 | tail -1
export GRAPH=1 CONTRACT=u8
for wh in "7680 4320" "3840 2160" "1920 1080" "15360 8640"; do set -- $wh; echo "-- u8 auto $1x$2"; W=$1 H=$2 BANDS=0 python tools/sweep.py; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/chk_bench.json 2>gpurun_out/chk_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/chk_bench.json"))
print(d["value"], d["roofline"]["frac"], d["variants"]["u8"]["us"], d["variants"]["detect_pad_clamp_abs"]["us"], d["e2e"]["ms_per_step"])
print(json.dumps(d["sizes"]))
PY
