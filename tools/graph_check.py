import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2305_00515_b200 import api
w, h = 1024, 256
d, pitch = api.alloc_input(w, h); api.synth_random_device(d, pitch, w, h, 1)
out, op = api.alloc_planes(w - 4, h - 4, ("gx",))
taps = api.make_stream_taps()
api.launch(d, pitch, w, h, taps, 1, out, op); torch.cuda.synchronize()
ref = out["gx"].clone()
out["gx"].zero_(); torch.cuda.synchronize()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    print("capturing on", s.cuda_stream, "status", torch.cuda.is_current_stream_capturing())
    api.launch(d, pitch, w, h, taps, 1, out, op, stream=s.cuda_stream)
torch.cuda.synchronize()
print("after capture, gx zero?", bool((out["gx"] == 0).all()))
g.replay(); torch.cuda.synchronize()
print("after replay equal ref?", bool(torch.equal(out["gx"], ref)))
