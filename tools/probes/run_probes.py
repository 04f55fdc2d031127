import ctypes as C, os, subprocess, sys
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "probes.so")
#
#
# load functions through the driver via torch's cuda python? use cupy-free path: cuda-python
from cuda.bindings import driver as cu
cu.cuInit(0)
torch.cuda.init(); torch.zeros(1, device="cuda")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-cubin", "-o",
                os.path.join(HERE, "probes.cubin"), os.path.join(HERE, "store_probe.cu")], check=True)
err, mod = cu.cuModuleLoad(os.path.join(HERE, "probes.cubin").encode())
err, f_store = cu.cuModuleGetFunction(mod, b"store_probe")
err, f_flat = cu.cuModuleGetFunction(mod, b"flat_probe")
import numpy as np
W, H = 7676, 4316
pitch = (W + 31) // 32 * 32
pl = [torch.empty((H, pitch), dtype=torch.int32, device="cuda") for _ in range(4)]
g = torch.empty((H, pitch), dtype=torch.float64, device="cuda")
def launch(fn, grid, block, args):
    # build kernel params: array of pointers to values
    vals = [np.array(v[0], dtype=v[1]) for v in args]
    ptrs = np.array([v.ctypes.data for v in vals], dtype=np.uint64)
    s = torch.cuda.current_stream().cuda_stream
    err, = cu.cuLaunchKernel(fn, *grid, *block, 0, s, ptrs.ctypes.data, 0)
    assert err == cu.CUresult.CUDA_SUCCESS, err
def timeit(fn, n=30):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
byts = W * H * 24
for band in (16, 32):
    for cs in (1, 0):
        args = [(p.data_ptr(), np.uint64) for p in pl] + [(g.data_ptr(), np.uint64), (pitch, np.int64),
                (W, np.int32), (H, np.int32), (band, np.int32), (cs, np.int32)]
        us = timeit(lambda: launch(f_store, ((W + 511) // 512, (H + band - 1) // band, 1), (128, 1, 1), args))
        print(f"store_probe band={band} cs={cs}: {us:.1f} us  {byts/us/1e3:.0f} GB/s")
flat = torch.empty(byts // 16 * 4, dtype=torch.int32, device="cuda")
us = timeit(lambda: launch(f_flat, (148 * 16, 1, 1), (256, 1, 1), [(flat.data_ptr(), np.uint64), (byts // 16, np.int64)]))
print(f"flat_probe: {us:.1f} us  {byts/us/1e3:.0f} GB/s")
