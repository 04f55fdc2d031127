cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
(python tools/layout_probe.py > gpurun_out/layout.txt 2>&1)
(CONTRACTS="sr u8" bash tools/variant_sweep.sh > gpurun_out/stq.txt 2>&1)
cat gpurun_out/layout.txt gpurun_out/stq.txt
