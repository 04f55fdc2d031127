#!/bin/bash
# g rebuilt on the host (SOBEL5_WIRE_G=1, default) vs g on the wire as f64:
# parity of the host paths, then the bench's e2e lines (8K C3, C4 frames)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -m pytest tests/test_gpu_wire16.py tests/test_gpu_frames.py tests/test_gpu_u8_only.py tests/test_gpu_sobel3.py -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do
for g in 1 0; do
  export SOBEL5_WIRE_G=$g
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/wg_$g.json 2>gpurun_out/wg_$g.err
  python - "$g" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/wg_{sys.argv[1]}.json").read().strip().splitlines()[-1])
e = d["e2e"]
print(f"WIRE_G={sys.argv[1]} value={d['value']:.1f} e2e={e['value']:.3f} {e['unit']} d2h={e['d2h_bytes_per_step']}",
      {k: v for k, v in e.items() if k not in ("value", "unit", "d2h_bytes_per_step", "h2d_bytes_per_step")})
PY
  python bench.py --steps 6 --warmup 3 --workload 1080p-batch --no-cpu-baseline > gpurun_out/wgc4_$g.json 2>gpurun_out/wgc4_$g.err
  python - "$g" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/wgc4_{sys.argv[1]}.json").read().strip().splitlines()[-1])
e = d["e2e"]
print(f"C4 WIRE_G={sys.argv[1]} value={d['value']:.1f} e2e={e['value']:.3f} {e['unit']} d2h={e['d2h_bytes_per_step']}")
PY
done
done
