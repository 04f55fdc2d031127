"""8K detect without padding (valid mode), both SaveModes, Python-loop timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_00515_b200 import api
w, h = 7680, 4320
ins = []
for i in range(4):
    d, pitch = api.alloc_input(w, h); api.synth_random_device(d, pitch, w, h, 1 + i); ins.append(d)
taps = api.make_stream_taps()
scratch = api.alloc_scratch(1, out_h=h, pitch=api.round_up(w, 32))
for mode in ("normalize", "clamp_abs"):
    out, op = api.alloc_planes(w - 4, h - 4, ("u8",))
    f = lambda i: api.detect_device(ins[i % 4], pitch, w, h, taps, 1, False, api.SaveMode[mode], out, op, scratch)
    for i in range(5): f(i)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for i in range(50): f(i)
    e1.record(); torch.cuda.synchronize()
    print("valid", mode, os.environ.get("SOBEL5_TMA_PLAIN_NARROW", "0"), round(e0.elapsed_time(e1) / 50 * 1e3, 1), "us")
