"""One 8K sobel5_run_host call twice (the host path: 32 row-chunk launches of the
gx..gdt int16 wire kernel, g rebuilt on the host) for ncu captures of the
wire kernel: ncu -k regex:sobel5_packed -s 40 -c 1 python tools/n16_capture.py"""
import ctypes as C, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2305_00515_b200 import _abi, api
w, h = 7680, 4320
ow, oh = w - 4, h - 4
ctx = api.Context(0); L = _abi.load(); taps = api.make_stream_taps()
h_in = torch.from_numpy(api.synth_random(w, h, 1)).pin_memory()
dt = {"gx": torch.int32, "gy": torch.int32, "gd": torch.int32, "gdt": torch.int32, "g": torch.float64}
h_out = {k: torch.empty((oh, ow), dtype=v, pin_memory=True) for k, v in dt.items()}
pl = _abi.Planes(pitch=ow)
for k, v in h_out.items(): setattr(pl, k, v.data_ptr())
d = _abi.Diag()
for _ in range(2):
    assert L.sobel5_run_host(ctx.handle, h_in.data_ptr(), w, h, C.byref(taps), 1, C.byref(pl), C.byref(d)) == 0
print("ok")
