#!/bin/bash
# int16 D2H wire: parity tests, then bench e2e with the wire on / off; 4K band re-sweep
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_wire16.py tests/test_gpu_host_paths.py tests/test_cpp_api.py tests/test_cpp_acceptance.py tests/test_gpu_dropin.py -m gpu -x -q 2>&1 | tail -3
for wire in 1 0 1 0; do
  SOBEL5_WIRE16=$wire python bench.py --steps 30 --warmup 5 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python - "$wire" <<'PY'
import json, sys
d = json.load(open("/tmp/b.json"))
e = d["e2e"]; c = d.get("e2e_cpp_api") or {}
print(f"wire={sys.argv[1]} value={d['value']:.1f} e2e={e['value']:.3f} Gpx/s {e['ms_per_step']:.2f} ms d2h={e['d2h_bytes_per_step']} cpp={c.get('value')} {c.get('ms_per_step')}")
PY
done
export GRAPH=1
echo "== 4K SR register ring bands 13,14,15,16"
SOBEL5_TMA_LOAD=0 W=3840 H=2160 BANDS=13,14,15,16 python tools/sweep.py
echo "== 4K SR default"
W=3840 H=2160 BANDS=0 python tools/sweep.py
