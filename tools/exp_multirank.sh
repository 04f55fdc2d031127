#!/bin/bash
# Multi-rank code path of bench.py on a one-GPU box (--share-gpu: all ranks on cuda:0, gloo)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531"
for wl in 8k 1080p-batch; do
  $R bench.py --gpus 2 --steps 20 --warmup 3 --workload $wl --share-gpu --no-cpu-baseline --no-e2e 2>gpurun_out/mr_$wl.err | tail -1 | cut -c1-400
done
for tr in peer gloo; do
  $R bench.py --gpus 2 --steps 10 --warmup 3 --workload 32k-bands --transport $tr --share-gpu --no-cpu-baseline --no-e2e 2>gpurun_out/mr_32k_$tr.err | tail -1 | cut -c1-400
done
$R bench.py --gpus 2 --steps 2 --warmup 1 --impl reference 2>/dev/null | tail -1 | cut -c1-300
