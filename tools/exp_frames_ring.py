"""8K end to end through the frames engine at n=1 (SOBEL5_FRAME_SLOTS x
SOBEL5_FRAME_CHUNKS: small staging rings may stay in the host LLC) against
sobel5_run_host; one subprocess per setting (the knobs are read per call)."""
import ctypes as C, os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1:
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    from paper_2305_00515_b200 import _abi, api
    w, h = 7680, 4320
    ow, oh = w - 4, h - 4
    ctx = api.Context(0)
    L = _abi.load()
    taps = api.make_stream_taps()
    h_in = torch.empty((h, w), dtype=torch.uint8, pin_memory=True)
    h_in.copy_(torch.from_numpy(api.synth_random(w, h, 1)))
    dt = {"gx": torch.int32, "gy": torch.int32, "gd": torch.int32, "gdt": torch.int32, "g": torch.float64}
    h_out = {k: torch.empty((oh, ow), dtype=v, pin_memory=True) for k, v in dt.items()}
    pl = _abi.Planes(pitch=ow)
    for k, v in h_out.items():
        setattr(pl, k, v.data_ptr())
    d = _abi.Diag()
    if sys.argv[1].startswith("run_host"):
        fn = lambda: L.sobel5_run_host(ctx.handle, h_in.data_ptr(), w, h, C.byref(taps), 1, C.byref(pl), C.byref(d))
    else:
        fn = lambda: L.sobel5_run_host_frames(ctx.handle, h_in.data_ptr(), w, h, 1, w * h, C.byref(taps), 1,
                                              C.byref(pl), ow * oh, C.byref(d))
    for _ in range(3):
        assert fn() == 0
    ts = []
    for i in range(20):
        t0 = time.perf_counter(); assert fn() == 0; ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{sys.argv[1]:28s} median {np.median(ts):6.2f} ms  min {np.min(ts):6.2f}", flush=True)
    sys.exit(0)
for rep in range(2):
    for c in (8, 16, 32):
        subprocess.run([sys.executable, __file__, f"run_host chunks {c}"],
                       env=dict(os.environ, SOBEL5_CHUNKS=str(c)))
    for chunks in (8, 16, 32, 64):
        for slots in (2, 4, 8):
            env = dict(os.environ, SOBEL5_FRAME_SLOTS=str(slots), SOBEL5_FRAME_CHUNKS=str(chunks))
            subprocess.run([sys.executable, __file__, f"frames chunks {chunks} slots {slots}"], env=env)
