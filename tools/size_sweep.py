"""Throughput vs image size (single image per launch, inputs rotated over
> L2 where they fit), SR and u8 contracts, 8-bit synthetic input."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_00515_b200 import api
taps = api.make_stream_taps()
print(f"{'size':>13s} {'contract':>8s} {'us':>9s} {'Gpx/s':>7s} {'GB/s':>6s} {'of 6544':>7s}")
for (w, h) in ((1920, 1080), (3840, 2160), (7680, 4320), (15360, 8640), (32768, 32768)):
    n_in = max(1, min(6, int(2 * 126e6 // (w * h)) + 1))
    ins = []
    for i in range(n_in):
        d, pitch = api.alloc_input(w, h); api.synth_random_device(d, pitch, w, h, 1 + i); ins.append(d)
    for contract, names, ob in (("sr", ("gx", "gy", "gd", "gdt", "g"), 24), ("u8", ("u8",), 1)):
        out, op = api.alloc_planes(w - 4, h - 4, names)
        for i in range(3): api.launch(ins[i % n_in], pitch, w, h, taps, 1, out, op)
        n = max(6, min(120, int(2e5 / (w * h / 4e6))))
        # a CUDA graph of n launches: the GPU time, not Python's launch rate
        # (a ctypes launch costs ~10 us of host time, more than a 1080p kernel)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            for i in range(n): api.launch(ins[i % n_in], pitch, w, h, taps, 1, out, op)
        graph.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); graph.replay(); e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / n * 1e3
        b = w * h + (w - 4) * (h - 4) * ob
        print(f"{w:6d}x{h:<6d} {contract:>8s} {us:9.1f} {w*h/us/1e3:7.1f} {b/us/1e3:6.0f} {b/us/1e3/6544:7.3f}", flush=True)
        del out, graph
        torch.cuda.empty_cache()
    del ins
    torch.cuda.empty_cache()
