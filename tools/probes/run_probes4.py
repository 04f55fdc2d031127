"""Store probe 4 (8 px per lane vs 4) at the 8K SR geometry."""
import os, subprocess
import numpy as np, torch
from cuda.bindings import driver as cu
HERE = os.path.dirname(os.path.abspath(__file__))
cub = "/tmp/p4.cubin"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-cubin", "-o", cub,
                os.path.join(HERE, "store_probe4.cu")], check=True)
torch.zeros(1, device="cuda")
err, mod = cu.cuModuleLoad(cub.encode())
def fn(name):
    e, f = cu.cuModuleGetFunction(mod, name.encode()); assert e == cu.CUresult.CUDA_SUCCESS, (name, e); return f
def launch(f, grid, block, args):
    vals = [np.array(v, dtype=t) for v, t in args]
    ptrs = np.array([v.ctypes.data for v in vals], dtype=np.uint64)
    e, = cu.cuLaunchKernel(f, *grid, *block, 0, torch.cuda.current_stream().cuda_stream, ptrs.ctypes.data, 0)
    assert e == cu.CUresult.CUDA_SUCCESS, e
def timeit(g, n=40):
    for _ in range(3): g()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n): g()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
W, H = 7676, 4316
pitch = (W + 63) // 64 * 64
byts = W * H * 24
pl = [torch.empty((H, pitch * 4), dtype=torch.uint8, device="cuda") for _ in range(4)]
g = torch.empty((H, pitch * 8), dtype=torch.uint8, device="cuda")
for px in (4, 8):
    f = fn(f"_Z6reg_pxILi{px}EEvPcS0_S0_S0_S0_liii")
    for band in (4, 8, 16, 32):
        args = [(p.data_ptr(), np.uint64) for p in pl] + [(g.data_ptr(), np.uint64), (pitch, np.int64),
                (W, np.int32), (H, np.int32), (band, np.int32)]
        cols = 128 * px
        us = timeit(lambda: launch(f, ((W + cols - 1) // cols, (H + band - 1) // band, 1), (128, 1, 1), args))
        print(f"px/lane={px} band={band:3d}: {us:6.1f} us {byts/us/1e3:5.0f} GB/s", flush=True)
f = fn("_Z8reg_pairPcS_S_S_S_liii")
for band in (4, 8, 16, 32):
    args = [(p.data_ptr(), np.uint64) for p in pl] + [(g.data_ptr(), np.uint64), (pitch, np.int64),
            (W, np.int32), (H, np.int32), (band, np.int32)]
    us = timeit(lambda: launch(f, ((W + 511) // 512, (H + band - 1) // band, 1), (128, 1, 1), args))
    print(f"pair-exchange band={band:3d}: {us:6.1f} us {byts/us/1e3:5.0f} GB/s", flush=True)
