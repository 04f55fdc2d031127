"""8K sobel5_run_host end to end (pinned buffers, g rebuilt on the host,
frame ring) over host-pool threads x ring chunks x slots; one subprocess per
setting (the knobs are read once per process)."""
import ctypes as C, itertools, os, subprocess, sys, time
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
    fn = lambda: L.sobel5_run_host(ctx.handle, h_in.data_ptr(), w, h, C.byref(taps), 1, C.byref(pl), C.byref(d))
    for _ in range(3):
        assert fn() == 0
    ts = []
    for i in range(30):
        t0 = time.perf_counter(); assert fn() == 0; ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{sys.argv[1]:34s} median {np.median(ts):6.2f} ms  min {np.min(ts):6.2f}", flush=True)
    sys.exit(0)
grid = [(16, ch, 4, 300, sp) for ch in (32, 64) for sp in ("mib", "pool")]
if os.environ.get("KNOB_GRID") == "chunks":  # DDIO-sized staging on host-memory-bound boxes
    grid = [(16, ch, sl, 300, 0) for ch, sl in ((32, 4), (48, 4), (64, 4), (96, 6), (128, 8), (24, 3))]
if os.environ.get("KNOB_GRID") == "threads":
    grid = [(th, ch, sl, 0, 1) for th, (ch, sl) in itertools.product((12, 14, 16), ((32, 4), (64, 4), (64, 6), (48, 4)))]
for rep in range(2):
    for th, ch, sl, sp, fd in grid:
        env = dict(os.environ, SOBEL5_HOST_THREADS=str(th), SOBEL5_FRAME_CHUNKS=str(ch),
                   SOBEL5_FRAME_SLOTS=str(sl), SOBEL5_POOL_SPIN_US=str(sp), SOBEL5_DECODE_SPLIT=str(fd))
        subprocess.run([sys.executable, __file__, f"threads {th} chunks {ch} slots {sl} spin {sp} split {fd}"],
                       env=env)
