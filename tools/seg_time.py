"""Stacked row band of C5 at N = 8 (32768 x 4096 body rows + 2-row halos above
and below, SR planes) timed with and without the TMA band rows
(SOBEL5_TMA_SEG=0/1); halos are local buffers here, a peer GPU's in C5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_00515_b200 import api

w, rows = 32768, 4096
body, pitch = api.alloc_input(w, rows)
api.synth_random_device(body, pitch, w, rows, 1)
top, _ = api.alloc_input(w, 2)
bot, _ = api.alloc_input(w, 2)
api.synth_random_device(top, pitch, w, 2, 2)
api.synth_random_device(bot, pitch, w, 2, 3)
out, op = api.alloc_planes(w - 4, rows, ("gx", "gy", "gd", "gdt", "g"))
taps = api.make_stream_taps()
res = {}
for rep in range(2):
    for tma in ("0", "1"):
        os.environ["SOBEL5_TMA_SEG"] = tma
        run = lambda: api.launch_band(top, body, bot, pitch, w, rows, taps, 1, out, op)
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(20):
            run()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        sig = tuple(float(out[k][:, :w - 4].double().sum()) for k in ("gx", "gd", "g"))
        res.setdefault("sig", sig)
        print(f"seg tma={tma} {us:7.1f} us  {w * (rows + 4) / us / 1e3:6.1f} Gpx/s  "
              f"same={res['sig'] == sig}", flush=True)
