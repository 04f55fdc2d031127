import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, torch, pyoracle
from paper_2305_00515_b200 import api
O = pyoracle.Oracle()
h, w = 9, 133
img = (np.random.default_rng(3).integers(0, 256, (h, w), dtype=np.uint8))
st_t = O.make_stream_taps(2, 3, 5, 7)
taps = api.Taps.from_dict(st_t.as_dict())
print(api.kernel_for(taps))
d, pitch = api.alloc_input(w, h); d[:, :w].copy_(torch.from_numpy(img))
out, op = api.alloc_planes(w - 4, h - 4, ("gx", "gy", "gd", "gdt"))
api.launch(d, pitch, w, h, taps, 1, out, op); torch.cuda.synchronize()
st, ref, _ = O.run_stream(img, st_t)
got = {k: v[:, :w-4].cpu().numpy() for k, v in out.items()}
for k in got:
    bad = np.argwhere(got[k] != ref[k])
    print(k, len(bad), bad[:12].tolist())
r, c = 0, slice(0, 12)
for k in got: print(k, got[k][r, c].tolist(), ref[k][r, c].tolist())
P = ref["gd"] + ref["gdt"]; M = ref["gd"] - ref["gdt"]
print("P", P[r, c].tolist()); print("M", M[r, c].tolist())
