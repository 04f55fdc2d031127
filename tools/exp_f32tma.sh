#!/bin/bash
# kernel F (packed FP32, taps beyond int16) with TMA band rows: parity, then band sweep vs the register ring
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -m pytest tests/test_gpu_f32.py tests/test_gpu_parity.py tests/test_gpu_stress.py -m gpu -x -q 2>&1 | tail -1
for prm in "2,3,5,7" "2,5,11,13"; do
  echo "== $prm ring"; SOBEL5_F32_TMA=0 PARAMS=$prm python tools/params_bench.py 2>/dev/null | grep "generic=0"
  for b in 0 4 6 8 12 16; do echo -n "tma band $b: "; SOBEL5_BAND=$b PARAMS=$prm python tools/params_bench.py 2>/dev/null | grep "generic=0"; done
done
