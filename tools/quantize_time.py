"""8K timing of the standalone device quantize (detail::quantize of a g plane)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_00515_b200 import api
w, h = 7676, 4316
g = torch.rand((h, w), dtype=torch.float64, device="cuda") * 3000
u8 = torch.empty((h, w), dtype=torch.uint8, device="cuda")
scratch = api.alloc_scratch(1)
for mode in ("clamp_abs", "normalize"):
    f = lambda: api.quantize_device(g, w, w, h, api.SaveMode[mode], u8, w, scratch)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize()
    print(mode, round(e0.elapsed_time(e1) / 20 * 1e3, 1), "us")
