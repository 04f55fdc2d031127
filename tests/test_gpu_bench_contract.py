"""GPU: bench.py's JSON contract, single rank and the multi-rank path
(torchrun, 2 ranks; --share-gpu puts both on cuda:0 over gloo so the N>1
code -- frame split, max over ranks, rank-0 line -- runs on a one-GPU box)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks")


def run(args, timeout=600):
    r = subprocess.run(args, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_single_rank_line(cuda):
    d = run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--no-cpu-baseline",
             "--no-e2e"])
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] == 5
    assert 0 < d["roofline"]["frac"] < 1.2 and d["roofline"]["bound"] == "hbm"


@pytest.mark.parametrize("workload", ["8k", "32k-bands"])
def test_two_ranks_share_gpu(cuda, workload):
    d = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
             "--master-addr", "127.0.0.1", "--master-port", "29537", "bench.py", "--gpus", "2",
             "--steps", "4", "--warmup", "3", "--workload", workload, "--share-gpu",
             "--no-cpu-baseline", "--no-e2e"])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["scaling"] == ("strong" if workload == "32k-bands" else "weak")


def test_two_ranks_e2e(cuda):
    """The e2e number at N > 1 is whole-job: every rank runs the host path on
    its own image, the time is the max over ranks."""
    d = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
             "--master-addr", "127.0.0.1", "--master-port", "29538", "bench.py", "--gpus", "2",
             "--steps", "4", "--warmup", "3", "--workload", "8k", "--share-gpu",
             "--no-cpu-baseline"])
    e = d["e2e"]
    assert e["ranks"] == 2 and e["value"] > 0
    assert e["h2d_bytes_per_step"] == 2 * 7680 * 4320
    # gx..gdt cross PCIe as int16 (the default-taps wire), the result planes
    # the caller receives are the full int32/f64 StreamResult
    assert e["d2h_bytes_per_step"] == 2 * 4 * 7680 * 4316 * 2  # int16 wire, g rebuilt on the host
    assert e["result_bytes_per_step"] == 2 * 7676 * 4316 * 24


def test_two_ranks_default_is_c5_with_e2e(cuda):
    """N > 1 defaults to the C5 strong-scaling workload (one 32768^2 image
    row-band partitioned, peer halos ordered by stream flags); e2e moves
    the band rows in and every output row out, max over ranks."""
    d = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
             "--master-addr", "127.0.0.1", "--master-port", "29539", "bench.py", "--gpus", "2",
             "--steps", "3", "--warmup", "3", "--share-gpu", "--no-cpu-baseline"], timeout=900)
    assert d["scaling"] == "strong" and "32768x32768" in d["config"]["workload"]
    assert d["timing"]["timed_as"] == "Python launch loop"
    e = d["e2e"]
    assert e["ranks"] == 2 and e["h2d_bytes_per_step"] == 32768 * 32768
    assert e["d2h_bytes_per_step"] >= 32764 * 32764 * 24
    assert d["cpu_baseline"] is None  # rank 0 at N=1 only
