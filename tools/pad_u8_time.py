import os, sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2305_00515_b200 import api
w, h = 7680, 4320
ins = []
for i in range(6):
    d, pitch = api.alloc_input(w, h); api.synth_random_device(d, pitch, w, h, 1 + i); ins.append(d)
out, op = api.alloc_planes(w, h, ("u8",))
taps = api.make_stream_taps()
f = lambda i: api.launch_ex(ins[i % 6], pitch, w, h, taps, 1, True, out, op)
for i in range(5): f(i)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
torch.cuda.synchronize(); e0.record()
for i in range(50): f(i)
e1.record(); torch.cuda.synchronize()
print("pad u8 tma_u8=", os.environ.get("SOBEL5_TMA_U8"), round(e0.elapsed_time(e1) / 50 * 1e3, 1), "us")
