"""Ablation of the paper's three ideas on B200 (8K, this library build):
prefetch ring on/off and the operator transformation on/off (SOBEL5_DENSE)
at runtime; the column-sharing variant is a compile-time build
(SOBEL5_COLSHARE, see tools/ablation.sh).  Every variant is checked
bit-exact against the oracle on a ragged image and against the default
variant's 8K planes (checksum) before it is timed."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np, torch, pyoracle
from paper_2305_00515_b200 import api

tag = os.environ.get("TAG", "default")
O = pyoracle.Oracle()
taps = api.make_stream_taps()
w, h = 7680, 4320
ins = []
for i in range(6):
    d, pitch = api.alloc_input(w, h); api.synth_random_device(d, pitch, w, h, 1 + i); ins.append(d)
SR = ("gx", "gy", "gd", "gdt", "g")


def check_small(pf):
    img = np.random.default_rng(5).integers(0, 256, (61, 517), dtype=np.uint8)
    d, p = api.alloc_input(517, 61); d[:, :517].copy_(torch.from_numpy(img))
    out, op = api.alloc_planes(513, 57, SR)
    api.launch(d, p, 517, 61, taps, pf, out, op); torch.cuda.synchronize()
    st, ref, _ = O.run_stream(img)
    return all(np.array_equal(out[k][:, :513].cpu().numpy(), ref[k]) for k in SR)


def run(contract, pf, dense):
    os.environ["SOBEL5_DENSE"] = "1" if dense else "0"
    names = SR if contract == "sr" else ("u8",)
    out, op = api.alloc_planes(w - 4, h - 4, names)
    ok = check_small(pf)
    api.launch(ins[0], pitch, w, h, taps, pf, out, op); torch.cuda.synchronize()
    sig = tuple(int(out[k][:, :w - 4].double().sum().item()) for k in names)
    for i in range(5): api.launch(ins[i % 6], pitch, w, h, taps, pf, out, op)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    N = 60
    for i in range(N): api.launch(ins[i % 6], pitch, w, h, taps, pf, out, op)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / N * 1e3
    b = w * h + (w - 4) * (h - 4) * (24 if contract == "sr" else 1)
    print(f"{tag:10s} {contract:3s} prefetch={pf} transform={'off' if dense else 'on ':3s} "
          f"{us:7.1f} us {w*h/us/1e3:6.1f} Gpx/s {b/us/1e3:6.0f} GB/s oracle_ok={ok} sig={hash(sig) & 0xffffffff:08x}",
          flush=True)
    os.environ["SOBEL5_DENSE"] = "0"


only = os.environ.get("ONLY")  # "sr,1,0" for the ncu pass
if only:
    c, pf, dn = only.split(","); run(c, int(pf), int(dn)); run(c, int(pf), int(dn))
else:
    for contract in ("sr", "u8"):
        run(contract, 1, 0)  # the design: shuffle + prefetch ring + operator transformation
        run(contract, 0, 0)  # Prefetch::off
        run(contract, 1, 1)  # dense 4 x 5x5 (no transformation), ring on
