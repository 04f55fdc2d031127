"""Run the 8K detect path (pad + normalize / clamp_abs) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_00515_b200 import api

w, h = int(os.environ.get("W", 7680)), int(os.environ.get("H", 4320))
mode = api.SaveMode[os.environ.get("MODE", "normalize")]
op = os.environ.get("OP", "5")
taps = api.make_stream_taps()
ins = []
for i in range(4):
    d, pitch = api.alloc_input(w, h)
    api.synth_random_device(d, pitch, w, h, 1 + i)
    ins.append(d)
out, opitch = api.alloc_planes(w, h, ("u8",))
scratch = api.alloc_scratch(1, out_h=h, pitch=opitch)
for i in range(int(os.environ.get("N", 6))):
    if op == "3":
        api.detect3_device(ins[i % 4], pitch, w, h, 1, True, mode, out, opitch, scratch)
    else:
        api.detect_device(ins[i % 4], pitch, w, h, taps, 1, True, mode, out, opitch, scratch)
torch.cuda.synchronize()
print("done")
