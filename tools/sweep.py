"""Kernel timing sweep over env knobs (SOBEL5_BAND, SOBEL5_PF, SOBEL5_GENERIC)."""
import itertools, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_00515_b200 import api

w, h = int(os.environ.get("W", 7680)), int(os.environ.get("H", 4320))
contract = os.environ.get("CONTRACT", "sr")
planes_names = {"sr": ("gx", "gy", "gd", "gdt", "g"), "u8": ("u8",), "int": ("gx", "gy", "gd", "gdt"),
                "sr3": ("gx", "gy", "g"), "sr32": ("gx", "gy", "gd", "gdt", "g32")}[contract]
outb = {"sr": 24, "u8": 1, "int": 16, "sr3": 16, "sr32": 20}[contract]
taps = api.make_stream_taps()
ins = []
for i in range(6):
    d, pitch = api.alloc_input(w, h)
    api.synth_random_device(d, pitch, w, h, 1 + i)
    ins.append(d)
out, op = api.alloc_planes(w - 4, h - 4, planes_names)
out3, op3 = api.alloc_planes(w - 2, h - 2, planes_names)
bands = [int(x) for x in os.environ.get("BANDS", "0").split(",")]
pfs = [0]  # (the CTAs-per-SM knob of an earlier build no longer exists)
res = {}
for band, pf in itertools.product(bands, pfs):
    os.environ["SOBEL5_BAND"] = str(band)
    k3 = os.environ.get("SOBEL3", "0") == "1"  # the 3x3 operator instead
    def go(i):
        if k3:
            api.launch3(ins[i % 6], pitch, w, h, 1, False, out3, op3)
        else:
            api.launch(ins[i % 6], pitch, w, h, taps, 1, out, op)
    for i in range(5):
        go(i)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    N = 60
    if os.environ.get("GRAPH", "0") == "1":  # device time without Python launch gaps
        torch.cuda.synchronize()
        gs = torch.cuda.Stream(); gs.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            for i in range(N):
                go(i)
        g.replay(); torch.cuda.synchronize()
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    else:
        torch.cuda.synchronize(); e0.record()
        for i in range(N):
            go(i)
        e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / N
    b = w * h + (w - 4) * (h - 4) * outb
    res[f"{band},{pf}"] = ms * 1e3
    print(f"band={band:4d} occ={pf} {ms*1e3:7.1f} us {w*h/ms/1e6:7.1f} Gpx/s {b/ms/1e6:6.0f} GB/s", flush=True)
