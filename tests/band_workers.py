"""Worker bodies for the multi-process row-band tests (spawned processes
import this module by name)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def _init(rank, world, port):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    return dist


def cpu_band_worker(rank, world, port, width, height, seed, result_dir):
    """Exchange halos with gloo on CPU tensors, then compute this band with the
    C oracle on [top; body; bot] and save it for the parent to compare."""
    import torch
    import pyoracle
    from paper_2305_00515_b200.bands import RowBandPartition, plan_bands
    dist = _init(rank, world, port)
    O = pyoracle.Oracle()
    img = O.synth_random(width, height, seed)
    plan = plan_bands(width, height, world, rank)
    pitch = width
    body = torch.from_numpy(img[plan.r0:plan.r1].copy())
    part = RowBandPartition(plan, body, pitch, transport="gloo")
    top, bot = part.exchange()
    stacked = [x.numpy() for x in (top, body, bot) if x is not None]
    st, out, _ = O.run_stream(np.concatenate(stacked, axis=0))
    assert st == 0
    assert out["gx"].shape[0] == plan.out_rows
    np.savez(os.path.join(result_dir, f"band{rank}.npz"), row0=plan.out_row0, **out)
    dist.barrier()
    dist.destroy_process_group()


def gpu_band_worker(rank, world, port, width, height, seed, transport, result_dir):
    """All ranks share cuda:0 (one GPU on the test box); control plane gloo.
    transport 'gloo' stages the halos through the host, 'peer' maps the
    neighbours' band buffers with CUDA IPC and reads the halos in-kernel."""
    import torch
    from paper_2305_00515_b200 import api
    from paper_2305_00515_b200.bands import RowBandPartition, plan_bands
    dist = _init(rank, world, port)
    torch.cuda.set_device(0)
    plan = plan_bands(width, height, world, rank)
    body, pitch = api.alloc_input(width, plan.body_rows, "cuda:0")
    api.synth_random_device(body, pitch, width, plan.body_rows, seed, row_offset=plan.r0)
    torch.cuda.synchronize()
    part = RowBandPartition(plan, body, pitch, transport=transport)
    planes, op = api.alloc_planes(width - 4, plan.out_rows, ("gx", "gy", "gd", "gdt", "g"),
                                  "cuda:0")
    dist.barrier()
    part.run(api.make_stream_taps(), planes, op)
    torch.cuda.synchronize()
    dist.barrier()  # neighbours must not free their bands before reads finish
    np.savez(os.path.join(result_dir, f"band{rank}.npz"), row0=plan.out_row0,
             **{k: v[:, : width - 4].cpu().numpy() for k, v in planes.items()})
    part.close()
    dist.barrier()
    dist.destroy_process_group()


def gpu_band_steps_worker(rank, world, port, width, height, steps, result_dir):
    """The peer transport over several steps with the band's input REWRITTEN
    before every step and no barrier between steps: the shared-page flags
    must order each rewrite after the neighbours' halo reads of the previous
    step, and each step's kernel after the neighbours' rewrites."""
    import torch
    from paper_2305_00515_b200 import api
    from paper_2305_00515_b200.bands import RowBandPartition, plan_bands
    dist = _init(rank, world, port)
    torch.cuda.set_device(0)
    plan = plan_bands(width, height, world, rank)
    body, pitch = api.alloc_input(width, plan.body_rows, "cuda:0")
    part = RowBandPartition(plan, body, pitch, transport="peer")
    stream = torch.cuda.Stream()
    outs = []
    for s in range(steps):
        planes, op = api.alloc_planes(width - 4, plan.out_rows, ("gx", "g"), "cuda:0")
        outs.append(planes)
    torch.cuda.synchronize()
    dist.barrier()  # setup done; no host synchronisation from here on
    for s in range(steps):
        api.synth_random_device(body, pitch, width, plan.body_rows, seed=50 + s,
                                row_offset=plan.r0, stream=stream.cuda_stream)
        part.run(api.make_stream_taps(), outs[s], op, stream=stream.cuda_stream)
    stream.synchronize()
    dist.barrier()  # neighbours must not free their bands before reads finish
    np.savez(os.path.join(result_dir, f"steps{rank}.npz"), row0=plan.out_row0,
             **{f"{k}{s}": outs[s][k][:, : width - 4].cpu().numpy()
                for s in range(steps) for k in ("gx", "g")})
    part.close()
    dist.barrier()
    dist.destroy_process_group()
