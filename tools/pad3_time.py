"""8K 3x3 replicate-padded launches (Stream3Result and u8), CUDA-graph timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_00515_b200 import api
w, h = 7680, 4320
ins = []
for i in range(6):
    d, pitch = api.alloc_input(w, h); api.synth_random_device(d, pitch, w, h, 1 + i); ins.append(d)
for names in (("gx", "gy", "g"), ("u8",)):
    out, op = api.alloc_planes(w, h, names)
    for i in range(5): api.launch3(ins[i % 6], pitch, w, h, 1, True, out, op)
    torch.cuda.synchronize()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream()); g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(40): api.launch3(ins[i % 6], pitch, w, h, 1, True, out, op, stream=s.cuda_stream)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    print("3x3 pad", "+".join(names), "tma_pad=", os.environ.get("SOBEL5_TMA_PAD", "1"),
          round(e0.elapsed_time(e1) / 40 * 1e3, 1), "us")
