"""GPU: sobel5_run_host_frames -- a stream of frames end to end through the
C ABI (run_stream per frame, pipelined across frames), every frame equal to
the oracle's run_stream (pipeline.hpp:452-477): the int16 wire (default
taps, StreamResult planes), other plane sets, pinned and pageable
destinations, padded frame strides, row-chunked large frames, custom and
fault-injected taps."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DT = {"gx": np.int32, "gy": np.int32, "gd": np.int32, "gdt": np.int32, "g": np.float64,
      "g32": np.float32, "u8": np.uint8}
SR = ("gx", "gy", "gd", "gdt", "g")


@pytest.fixture(scope="module")
def ctx(cuda):
    from paper_2305_00515_b200 import api
    c = api.Context(0)
    yield c
    c.close()


def run_frames(ctx, frames, planes, taps, pinned, in_pad=0, out_pad=0, status=0):
    import torch
    from paper_2305_00515_b200 import _abi
    L = _abi.load()
    n = len(frames)
    h, w = frames[0].shape
    ow, oh = w - 4, h - 4
    in_stride = h * w + in_pad
    buf = np.zeros(n * in_stride, np.uint8)
    for f, img in enumerate(frames):
        buf[f * in_stride: f * in_stride + h * w] = img.reshape(-1)
    out_stride = ow * oh + out_pad
    res = {k: np.full(n * out_stride, 7, DT[k]) for k in planes}
    if pinned:
        res = {k: torch.from_numpy(v).pin_memory() for k, v in res.items()}
        buf_t = torch.from_numpy(buf).pin_memory()
        src = buf_t.data_ptr()
    else:
        src = buf.ctypes.data
    pl = _abi.Planes(pitch=ow)
    for k, v in res.items():
        setattr(pl, k, v.data_ptr() if pinned else v.ctypes.data)
    d = _abi.Diag()
    st = L.sobel5_run_host_frames(ctx.handle, src, w, h, n, in_stride, C.byref(taps), 1,
                                  C.byref(pl), out_stride, C.byref(d))
    assert st == status, st
    out = {}
    for k, v in res.items():
        a = v.numpy() if pinned else v
        out[k] = [a[f * out_stride: f * out_stride + ow * oh].reshape(oh, ow) for f in range(n)]
        if out_pad:  # the gaps between frames stay untouched
            for f in range(n):
                assert np.all(a[f * out_stride + ow * oh: (f + 1) * out_stride] == 7)
    return out, d, L.sobel5_ctx_last_d2h_bytes(ctx.handle)


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("h,w,n", [(5, 5, 3), (61, 97, 7), (300, 517, 5), (2100, 2060, 3)])
def test_frames_sr_wire(ctx, oracle, pinned, h, w, n):
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(h * w + n)
    frames = [rng.integers(0, 256, (h, w), dtype=np.uint8) & (0xFF if f % 2 else 0x0F)
              for f in range(n)]
    out, d, d2h = run_frames(ctx, frames, SR, api.make_stream_taps(), pinned, in_pad=3, out_pad=5)
    for f, img in enumerate(frames):
        st, ref, _ = oracle.run_stream(img)
        assert st == 0
        for k in SR:
            np.testing.assert_array_equal(out[k][f], ref[k], err_msg=f"frame {f} {k}")
    ow, oh = w - 4, h - 4
    dp = (ow + 31) // 32 * 32
    assert d2h == n * 4 * dp * oh * 2  # the int16 wire, g rebuilt on the host


@pytest.mark.parametrize("planes", [("gx", "u8"), ("g32", "gd"), SR + ("u8",), ("g",)])
def test_frames_other_planes(ctx, oracle, planes):
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(len(planes))
    frames = [rng.integers(0, 256, (130, 259), dtype=np.uint8) & 0x07 for _ in range(6)]
    out, d, _ = run_frames(ctx, frames, planes, api.make_stream_taps(), pinned=False)
    for f, img in enumerate(frames):
        st, ref, _ = oracle.run_stream(img)
        for k in planes:
            if k == "u8":
                np.testing.assert_array_equal(out[k][f], oracle.clamp_abs(ref["g"]))
            elif k == "g32":
                exact = ref["g"].astype(np.float32)
                ulps = np.abs(out[k][f].view(np.int32).astype(np.int64) - exact.view(np.int32))
                assert ulps.max() <= 1
            else:
                np.testing.assert_array_equal(out[k][f], ref[k], err_msg=f"frame {f} {k}")


def test_frames_custom_and_fault_taps(ctx, oracle, reference):
    from paper_2305_00515_b200 import _abi, api
    rng = np.random.default_rng(3)
    frames = [rng.integers(0, 256, (97, 301), dtype=np.uint8) for _ in range(4)]
    t = oracle.make_stream_taps(2, 3, 5, 7)
    out, d, _ = run_frames(ctx, frames, SR, api.Taps.from_dict(t.as_dict()), pinned=True)
    for f, img in enumerate(frames):
        st, ref, _ = oracle.run_stream(img, t)
        for k in SR:
            np.testing.assert_array_equal(out[k][f], ref[k], err_msg=f"frame {f} {k}")
    # odd fault in the second frame only: ParityViolation, the first odd pixel's pair
    code, tf, msg = reference.make_stream_taps(1, 1, 1, 1)
    tf.k1[2] += 1
    flat = [np.zeros((97, 301), np.uint8), frames[1], frames[2]]
    _, d, _ = run_frames(ctx, flat, SR, api.Taps.from_dict(tf.as_dict()), pinned=False,
                         status=_abi.PARITY_VIOLATION)
    assert d.violations > 0
    code, _, _, want = reference.run_stream(frames[1], tf, lanes=301, prefetch=True, workers=1)
    assert code == 17 and want == f"odd sum/difference pair ({d.sum}, {d.diff})"


def test_frames_errors(ctx):
    from paper_2305_00515_b200 import _abi, api
    L = _abi.load()
    taps = api.make_stream_taps()
    img = np.zeros(10 * 10, np.uint8)
    res = np.zeros(6 * 6, np.int32)
    pl = _abi.Planes(pitch=6)
    pl.gx = res.ctypes.data
    d = _abi.Diag()
    assert L.sobel5_run_host_frames(ctx.handle, img.ctypes.data, 4, 10, 1, 40, C.byref(taps), 1,
                                    C.byref(pl), 36, C.byref(d)) == _abi.IMAGE_TOO_SMALL
    assert L.sobel5_run_host_frames(ctx.handle, img.ctypes.data, 10, 10, 1, 99, C.byref(taps), 1,
                                    C.byref(pl), 36, C.byref(d)) == _abi.INVALID_ARG  # stride < W*H
    assert L.sobel5_run_host_frames(ctx.handle, img.ctypes.data, 10, 10, 0, 100, C.byref(taps), 1,
                                    C.byref(pl), 36, C.byref(d)) == _abi.INVALID_ARG
    assert L.sobel5_run_host_frames(ctx.handle, img.ctypes.data, 10, 10, 1, 100, C.byref(taps), 1,
                                    C.byref(pl), 36, C.byref(d)) == 0


def test_frames_python_api(ctx, oracle):
    """Context.run_host_frames (the Python face of the C call), u8 included."""
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(11)
    frames = rng.integers(0, 256, (5, 70, 133), dtype=np.uint8)
    st, res, d = ctx.run_host_frames(frames, api.make_stream_taps(), planes=SR + ("u8",))
    assert st == 0 and d.violations == 0
    for f in range(5):
        _, ref, _ = oracle.run_stream(frames[f])
        for k in SR:
            np.testing.assert_array_equal(res[k][f], ref[k], err_msg=f"frame {f} {k}")
        np.testing.assert_array_equal(res["u8"][f], oracle.clamp_abs(ref["g"]))


def test_frames_parity_pair_is_the_first_frames(ctx, reference):
    """A stream of frames stops at the first frame with an odd pair, as a loop
    of run_stream calls would: frame 1's first pair is reported although
    frame 2 has one at an earlier strip and row."""
    from paper_2305_00515_b200 import _abi, api
    rng = np.random.default_rng(4)
    h, w, lanes = 120, 301, 64
    frames = [np.zeros((h, w), np.uint8) for _ in range(3)]
    frames[1][60:70, 130:160] = rng.integers(0, 256, (10, 30), dtype=np.uint8)  # strip 2, rows ~56..
    frames[2][3:9, 5:50] = rng.integers(0, 256, (6, 45), dtype=np.uint8)         # strip 0, rows ~0..
    code, t, msg = reference.make_stream_taps(1, 1, 1, 1)
    t.k1[2] += 1
    L = _abi.load()
    assert L.sobel5_ctx_set_strip_width(ctx.handle, lanes - 4) == 0
    try:
        _, d, _ = run_frames(ctx, frames, SR, api.Taps.from_dict(t.as_dict()), pinned=False,
                             status=_abi.PARITY_VIOLATION)
    finally:
        L.sobel5_ctx_set_strip_width(ctx.handle, 0)
    code, _, _, want = reference.run_stream(frames[1], t, lanes=lanes, prefetch=True, workers=1)
    assert code == 17 and want == f"odd sum/difference pair ({d.sum}, {d.diff})"


@pytest.mark.parametrize("seed", range(8))
def test_host_paths_random_shapes(ctx, oracle, seed):
    """Random frame shapes / counts / strides / pinnedness through the frames
    engine and sobel5_run_host (both on the wire with g rebuilt on the host):
    every plane equals the oracle's."""
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(100 + seed)
    h = int(rng.integers(5, 1400))
    w = int(rng.integers(5, 1400))
    n = int(rng.integers(1, 4))
    frames = [rng.integers(0, 256, (h, w), dtype=np.uint8) for _ in range(n)]
    out, d, _ = run_frames(ctx, frames, SR, api.make_stream_taps(), pinned=bool(seed % 2),
                           in_pad=int(rng.integers(0, 9)), out_pad=int(rng.integers(0, 9)))
    for f, img in enumerate(frames):
        _, ref, _ = oracle.run_stream(img)
        for k in SR:
            np.testing.assert_array_equal(out[k][f], ref[k], err_msg=f"frames {h}x{w} frame {f} {k}")
        st, res, _ = ctx.run_host(img, api.make_stream_taps())
        assert st == 0
        for k in SR:
            np.testing.assert_array_equal(res[k], ref[k], err_msg=f"run_host {h}x{w} {k}")
