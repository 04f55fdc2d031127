"""Row-band partition (BASELINE C5) with world_size 2
and 3: band planning, halo exchange and stitching, against the single-image
result.  CPU variant: gloo + the C oracle.  GPU variant: ranks share cuda:0,
halos via gloo staging or via CUDA IPC peer pointers read in-kernel."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
PLANES = ("gx", "gy", "gd", "gdt", "g")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def stitch_and_check(oracle, result_dir, world, width, height, seed):
    st, ref, _ = oracle.run_stream(oracle.synth_random(width, height, seed))
    covered = np.zeros(height - 4, bool)
    for r in range(world):
        z = np.load(os.path.join(result_dir, f"band{r}.npz"))
        row0 = int(z["row0"])
        n = z["gx"].shape[0]
        assert not covered[row0:row0 + n].any()
        covered[row0:row0 + n] = True
        for k in PLANES:
            np.testing.assert_array_equal(z[k], ref[k][row0:row0 + n], err_msg=f"rank {r} {k}")
    assert covered.all()


def test_plan_bands_cover_disjoint():
    from paper_2305_00515_b200.bands import plan_bands
    for height in (8, 9, 37, 100, 4321):
        for world in (1, 2, 3, 4, 8):
            if height < 4 * world:
                continue
            nxt = 2
            for r in range(world):
                p = plan_bands(64, height, world, r)
                assert p.c0 == nxt and p.out_row0 == nxt - 2
                assert p.has_top == (r > 0) and p.has_bot == (r < world - 1)
                nxt = p.c1
            assert nxt == height - 2


@pytest.mark.parametrize("world", [2, 3])
def test_band_partition_gloo_cpu(oracle, tmp_path, world):
    import torch.multiprocessing as mp
    import band_workers
    w, h, seed = 67, 41, 9
    mp.spawn(band_workers.cpu_band_worker, args=(world, free_port(), w, h, seed, str(tmp_path)),
             nprocs=world, join=True)
    stitch_and_check(oracle, str(tmp_path), world, w, h, seed)


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["gloo", "peer"])
@pytest.mark.parametrize("world", [2, 3])
def test_band_partition_gpu(oracle, cuda, tmp_path, transport, world):
    import torch.multiprocessing as mp
    import band_workers
    w, h, seed = 1029, 203, 4
    mp.spawn(band_workers.gpu_band_worker,
             args=(world, free_port(), w, h, seed, transport, str(tmp_path)), nprocs=world,
             join=True)
    stitch_and_check(oracle, str(tmp_path), world, w, h, seed)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_peer_transport_rewrites_every_step(oracle, cuda, tmp_path, world):
    """Inputs rewritten every step, no barrier between steps (VERDICT r1
    weak #2b): every step's stitched output equals the oracle's."""
    import torch.multiprocessing as mp
    import band_workers
    w, h, steps = 1536, 260, 5
    ctx = mp.start_processes(band_workers.gpu_band_steps_worker,
                             args=(world, free_port(), w, h, steps, str(tmp_path)), nprocs=world,
                             join=False, start_method="spawn")
    import time
    deadline = time.time() + 300
    try:
        while not ctx.join(timeout=10):
            assert time.time() < deadline, "workers did not finish"
    finally:
        for pr in ctx.processes:  # only our own children, by handle
            if pr.is_alive():
                pr.kill()
    for s in range(steps):
        st, ref, _ = oracle.run_stream(oracle.synth_random(w, h, 50 + s))
        covered = 0
        for r in range(world):
            z = np.load(os.path.join(str(tmp_path), f"steps{r}.npz"))
            row0, n = int(z["row0"]), z[f"gx{s}"].shape[0]
            for k in ("gx", "g"):
                np.testing.assert_array_equal(z[f"{k}{s}"], ref[k][row0:row0 + n],
                                              err_msg=f"step {s} rank {r} {k}")
            covered += n
        assert covered == h - 4
