import ctypes as C, os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2305_00515_b200 import _abi, api
w, h = 7680, 4320
ow, oh = w - 4, h - 4
ctx = api.Context(0)
L = _abi.load()
taps = api.make_stream_taps()
h_in = torch.empty((h, w), dtype=torch.uint8, pin_memory=True)
h_in.copy_(torch.from_numpy(api.synth_random(w, h, 1)))
dt = {"gx": torch.int32, "gy": torch.int32, "gd": torch.int32, "gdt": torch.int32, "g": torch.float64}
h_out = {k: torch.empty((oh, ow), dtype=v, pin_memory=True) for k, v in dt.items()}
pl = _abi.Planes(pitch=ow)
for k, v in h_out.items():
    setattr(pl, k, v.data_ptr())
d = _abi.Diag()
for name, fn in (("run_host", lambda: L.sobel5_run_host(ctx.handle, h_in.data_ptr(), w, h, C.byref(taps), 1, C.byref(pl), C.byref(d))),
                 ("frames n=1", lambda: L.sobel5_run_host_frames(ctx.handle, h_in.data_ptr(), w, h, 1, w * h, C.byref(taps), 1, C.byref(pl), ow * oh, C.byref(d)))) * 2:
    fn()
    ts = []
    for i in range(20):
        t0 = time.perf_counter(); assert fn() == 0; ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name}: median {np.median(ts):.2f} ms  min {np.min(ts):.2f}")
