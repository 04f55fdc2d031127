lscpu | grep -E "Model name|^CPU\(s\)|Thread|NUMA node\(s\)|L3" > gpurun_out/host.txt; free -g >> gpurun_out/host.txt; cat /sys/kernel/mm/transparent_hugepage/enabled >> gpurun_out/host.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$? >> gpurun_out/bench.err
python tools/pcie_probe.py > gpurun_out/pcie.txt 2>&1
N=40 python tools/e2e_trace.py > gpurun_out/e2e_trace.txt 2>&1
echo done
