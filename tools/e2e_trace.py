"""Per-call wall time of sobel5_run_host (8K SR, pinned planes, int16 wire) over many calls."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
ts = []
for i in range(int(os.environ.get("N", "80"))):
    t0 = time.perf_counter()
    st = L.sobel5_run_host(ctx.handle, h_in.data_ptr(), w, h, C.byref(taps), 1, C.byref(pl), C.byref(d))
    ts.append((time.perf_counter() - t0) * 1e3)
    assert st == 0
ts = np.array(ts)
print("first 10:", np.round(ts[:10], 2))
print("last 10:", np.round(ts[-10:], 2))
for a in range(0, len(ts), 10):
    print(f"calls {a:3d}-{a+9:3d}: median {np.median(ts[a:a+10]):.2f} ms")
