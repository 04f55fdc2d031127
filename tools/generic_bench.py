"""Time the generic-taps kernel (non-default FilterParams) at 8K, SR and u8."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_00515_b200 import api

w, h = 7680, 4320
ins = []
for i in range(8):
    d, pitch = api.alloc_input(w, h)
    api.synth_random_device(d, pitch, w, h, seed=10 + i)
    ins.append(d)
for params in [(1, 2, 6, 4), (1, 1, 1, 1), (2, 3, 5, 7), (1, 32768, 1, 1)]:
    taps = api.make_stream_taps(api.FilterParams(*params))
    for planes, nb in ((("gx", "gy", "gd", "gdt", "g"), 24), (("u8",), 1)):
        out, op = api.alloc_planes(w - 4, h - 4, planes)
        for i in range(3):
            api.launch(ins[i % 8], pitch, w, h, taps, 1, out, op)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize(); e0.record()
        N = 30
        for i in range(N):
            api.launch(ins[i % 8], pitch, w, h, taps, 1, out, op)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / N * 1e3
        print(f"{params} {'sr' if nb == 24 else 'u8'}: {us:.1f} us {(w*h + (w-4)*(h-4)*nb)/us/1e3:.0f} GB/s", flush=True)
        del out
