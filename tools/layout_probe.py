"""Output-plane layout probe for the SR contract at 8K: does the placement of
the five StreamResult planes in HBM (base offsets between planes, row pitch
padding) change the write throughput of the packed kernel?

Planes are carved from one allocation: plane i starts at i * (plane_bytes +
DELTA) bytes (rounded to 256 B), every plane with pitch round_up(out_w, 32) +
EXTRA elements.  Prints one line per (delta, extra)."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_00515_b200 import api  # noqa: E402

w, h = int(os.environ.get("W", 7680)), int(os.environ.get("H", 4320))
ow, oh = w - 4, h - 4
taps = api.make_stream_taps()
ins = []
for i in range(6):
    d, pitch = api.alloc_input(w, h)
    api.synth_random_device(d, pitch, w, h, 1 + i)
    ins.append(d)
names = ("gx", "gy", "gd", "gdt", "g")
esz = {"gx": 4, "gy": 4, "gd": 4, "gdt": 4, "g": 8}
deltas = [int(x) for x in os.environ.get("DELTAS", "0,256,1024,4096,8192,30720,65536,1048576").split(",")]
extras = [int(x) for x in os.environ.get("EXTRAS", "0,4,8,32,64").split(",")]
N = int(os.environ.get("N", 60))
ref = None
for delta, extra in itertools.product(deltas, extras):
    op = api.round_up(ow, 32) + extra
    sizes = [op * oh * esz[k] for k in names]
    offs, cur = [], 0
    for s in sizes:
        offs.append(cur)
        cur = (cur + s + delta + 255) // 256 * 256
    buf = torch.empty(cur + 4096, dtype=torch.uint8, device="cuda")
    base = (buf.data_ptr() + 255) // 256 * 256 - buf.data_ptr()
    planes = {}
    for k, o, s in zip(names, offs, sizes):
        t = buf[base + o: base + o + s]
        planes[k] = t.view(torch.float64 if k == "g" else torch.int32).view(oh, op)
    for i in range(5):
        api.launch(ins[i % 6], pitch, w, h, taps, 1, planes, op)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(N):
        api.launch(ins[i % 6], pitch, w, h, taps, 1, planes, op)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / N
    b = w * h + ow * oh * 24
    chk = int(planes["gx"][:, :ow].sum().item()) ^ int(planes["gd"][:, :ow].sum().item())
    if ref is None:
        ref = chk
    print(f"delta={delta:8d} extra={extra:3d} pitch={op} {ms*1e3:7.1f} us "
          f"{b/ms/1e6:6.0f} GB/s{'' if chk == ref else ' MISMATCH'}", flush=True)
    del planes, buf
    torch.cuda.empty_cache()
