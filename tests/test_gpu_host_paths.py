"""GPU: the host-buffer entry points behind run_stream (sobel5_ctx.cu).

Pageable destinations go through pinned staging plus a host thread pool,
page-locked ones are DMA'd directly, and the split begin/finish form lets
the C++ run_stream build its result planes while the device works.  Every
path must produce the same planes as the oracle; misuse is rejected without
leaving the context unusable."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PLANES = ("gx", "gy", "gd", "gdt", "g")
DT = {"gx": np.int32, "gy": np.int32, "gd": np.int32, "gdt": np.int32, "g": np.float64,
      "g32": np.float32, "u8": np.uint8}
BIT = {"gx": 1, "gy": 2, "gd": 4, "gdt": 8, "g": 16, "g32": 32, "u8": 64}


@pytest.fixture(scope="module")
def ctx(cuda):
    from paper_2305_00515_b200 import api
    c = api.Context(0)
    yield c
    c.close()


def planes_struct(res, ow):
    from paper_2305_00515_b200 import _abi
    pl = _abi.Planes(pitch=ow)
    for k, v in res.items():
        setattr(pl, k, v.data_ptr() if hasattr(v, "data_ptr") else v.ctypes.data)
    return pl


@pytest.mark.parametrize("h,w", [(5, 5), (61, 97), (300, 1030), (1100, 2051)])
def test_pageable_and_pinned_destinations(ctx, oracle, h, w):
    import torch
    from paper_2305_00515_b200 import _abi, api
    img = np.random.default_rng(h + w).integers(0, 256, (h, w), dtype=np.uint8)
    if w % 2:
        img &= 0x0F
    st, ref, _ = oracle.run_stream(img)
    assert st == 0
    ow, oh = w - 4, h - 4
    taps = api.make_stream_taps()
    L = _abi.load()
    # pageable numpy planes + pageable input
    res = {k: np.full((oh, ow), 7, DT[k]) for k in PLANES + ("u8",)}
    d = _abi.Diag()
    assert L.sobel5_run_host(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1,
                             C.byref(planes_struct(res, ow)), C.byref(d)) == 0
    for k in PLANES:
        np.testing.assert_array_equal(res[k], ref[k], err_msg=f"pageable {k}")
    np.testing.assert_array_equal(res["u8"], oracle.clamp_abs(ref["g"]))
    # pinned planes and pinned input, mixed with one pageable plane
    h_in = torch.from_numpy(img).pin_memory()
    pin = {k: torch.full((oh, ow), 7, dtype=getattr(torch, np.dtype(DT[k]).name)).pin_memory()
           for k in ("gx", "gd", "g")}
    page = {k: np.full((oh, ow), 7, DT[k]) for k in ("gy", "gdt")}
    pl = planes_struct(pin, ow)
    for k, v in page.items():
        setattr(pl, k, v.ctypes.data)
    assert L.sobel5_run_host(ctx.handle, h_in.data_ptr(), w, h, C.byref(taps), 0, C.byref(pl),
                             C.byref(d)) == 0
    for k, v in pin.items():
        np.testing.assert_array_equal(v.numpy(), ref[k], err_msg=f"pinned {k}")
    for k, v in page.items():
        np.testing.assert_array_equal(v, ref[k], err_msg=f"mixed pageable {k}")


def test_begin_finish(ctx, oracle):
    from paper_2305_00515_b200 import _abi, api
    L = _abi.load()
    h, w = 777, 1301
    img = np.random.default_rng(9).integers(0, 256, (h, w), dtype=np.uint8) & 0x07
    st, ref, _ = oracle.run_stream(img)
    ow, oh = w - 4, h - 4
    taps = api.make_stream_taps()
    want = ("gx", "gdt", "g", "u8")
    mask = sum(BIT[k] for k in want)
    assert L.sobel5_run_host_begin(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1, mask) == 0
    # a second begin or a run_host while one is pending is refused
    assert L.sobel5_run_host_begin(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1,
                                   mask) == _abi.INVALID_ARG
    res = {k: np.zeros((oh, ow), DT[k]) for k in want}
    d = _abi.Diag()
    assert L.sobel5_run_host(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1,
                             C.byref(planes_struct(res, ow)), C.byref(d)) == _abi.INVALID_ARG
    assert L.sobel5_run_host_finish(ctx.handle, C.byref(planes_struct(res, ow)), C.byref(d)) == 0
    for k in ("gx", "gdt", "g"):
        np.testing.assert_array_equal(res[k], ref[k], err_msg=k)
    np.testing.assert_array_equal(res["u8"], oracle.clamp_abs(ref["g"]))
    # finish without begin; planes not matching the mask (the pending work
    # is still completed and the context stays usable)
    assert L.sobel5_run_host_finish(ctx.handle, C.byref(planes_struct(res, ow)),
                                    C.byref(d)) == _abi.INVALID_ARG
    assert L.sobel5_run_host_begin(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1, mask) == 0
    part = {k: res[k] for k in ("gx", "g")}
    assert L.sobel5_run_host_finish(ctx.handle, C.byref(planes_struct(part, ow)),
                                    C.byref(d)) == _abi.INVALID_ARG
    assert L.sobel5_run_host_begin(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1,
                                   0) == _abi.INVALID_ARG
    assert L.sobel5_run_host_begin(ctx.handle, img.ctypes.data, 4, h, C.byref(taps), 1,
                                   mask) == _abi.IMAGE_TOO_SMALL
    res2 = {k: np.zeros((oh, ow), DT[k]) for k in want}
    assert L.sobel5_run_host(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1,
                             C.byref(planes_struct(res2, ow)), C.byref(d)) == 0
    for k in want:
        np.testing.assert_array_equal(res2[k], res[k])


def test_begin_finish_parity_violation(ctx):
    """Fault-injected taps: finish reports the odd pair like run_host."""
    from paper_2305_00515_b200 import _abi, api
    L = _abi.load()
    taps = api.make_stream_taps()
    taps.k0[0] += 1
    img = np.random.default_rng(4).integers(0, 256, (40, 70), dtype=np.uint8)
    assert L.sobel5_run_host_begin(ctx.handle, img.ctypes.data, 70, 40, C.byref(taps), 1,
                                   0x1F) == 0
    res = {k: np.zeros((36, 66), DT[k]) for k in PLANES}
    d = _abi.Diag()
    assert L.sobel5_run_host_finish(ctx.handle, C.byref(planes_struct(res, 66)),
                                    C.byref(d)) == _abi.PARITY_VIOLATION
    assert d.violations > 0


def test_chunk_staging_consumer(ctx, oracle):
    """begin -> _chunk/_staging (consume rows as they land) -> finish(NULL)."""
    from paper_2305_00515_b200 import _abi, api
    L = _abi.load()
    h, w = 2300, 517
    img = np.random.default_rng(21).integers(0, 256, (h, w), dtype=np.uint8) & 0x0F
    st, ref, _ = oracle.run_stream(img)
    ow, oh = w - 4, h - 4
    taps = api.make_stream_taps()
    assert L.sobel5_run_host_staging(ctx.handle, 0) is None  # nothing pending
    assert L.sobel5_run_host_begin(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1,
                                   BIT["gd"] | BIT["g"]) == 0
    assert L.sobel5_run_host_staging(ctx.handle, 0) is None  # gx not in the mask
    got = {}
    for k, i in (("gd", 2), ("g", 4)):
        p = L.sobel5_run_host_staging(ctx.handle, i)
        assert p
        got[k] = (p, np.dtype(DT[k]))
    y0, y1 = C.c_int(), C.c_int()
    rows, k = [], 0
    while L.sobel5_run_host_chunk(ctx.handle, k, C.byref(y0), C.byref(y1)) == 0:
        rows.append((y0.value, y1.value))
        k += 1
    assert rows[0][0] == 0 and rows[-1][1] == oh and len(rows) > 1
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    for name, (p, dt) in got.items():
        buf = (C.c_char * (ow * oh * dt.itemsize)).from_address(p)
        arr = np.frombuffer(buf, dtype=dt).reshape(oh, ow).copy()
        np.testing.assert_array_equal(arr, ref[name], err_msg=name)
    d = _abi.Diag()
    assert L.sobel5_run_host_finish(ctx.handle, None, C.byref(d)) == 0
    assert L.sobel5_run_host_chunk(ctx.handle, 0, C.byref(y0), C.byref(y1)) == _abi.INVALID_ARG


def test_sobel3_begin_finish(ctx, oracle):
    """The 3x3 split form: sobel3_run_host_begin -> finish, pageable planes."""
    from paper_2305_00515_b200 import _abi
    L = _abi.load()
    h, w = 1200, 301
    img = np.random.default_rng(31).integers(0, 256, (h, w), dtype=np.uint8)
    st, ref = oracle.sobel3_2d(img)
    assert st == 0
    ow, oh = w - 2, h - 2
    assert L.sobel3_run_host_begin(ctx.handle, img.ctypes.data, w, h, 1,
                                   BIT["gx"] | BIT["gd"]) == _abi.INVALID_ARG  # no gd for 3x3
    assert L.sobel3_run_host_begin(ctx.handle, img.ctypes.data, 2, h, 1,
                                   BIT["gx"]) == _abi.IMAGE_TOO_SMALL
    want = ("gx", "gy", "g", "u8")
    assert L.sobel3_run_host_begin(ctx.handle, img.ctypes.data, w, h, 1,
                                   sum(BIT[k] for k in want)) == 0
    res = {k: np.zeros((oh, ow), DT[k]) for k in want}
    d = _abi.Diag()
    assert L.sobel5_run_host_finish(ctx.handle, C.byref(planes_struct(res, ow)), C.byref(d)) == 0
    for k in ("gx", "gy", "g"):
        np.testing.assert_array_equal(res[k], ref[k], err_msg=k)
    np.testing.assert_array_equal(res["u8"], oracle.quantize(ref["g"], "clamp_abs"))


def test_python_oracle_mirrors(ctx, oracle):
    """api.sobel5_4d / api.diag_via_sum_diff (oracle.hpp mirrors on the GPU)."""
    from paper_2305_00515_b200 import api
    img = api.synth_random(131, 47, 5)
    for prm in ((1, 2, 6, 4), (2, 3, 5, 7)):
        p = api.FilterParams(*prm)
        st, ref, _ = oracle.run_stream(img, oracle.make_stream_taps(*prm))
        r = api.sobel5_4d(img, p)
        for k in ("gx", "gy", "gd", "gdt", "g"):
            np.testing.assert_array_equal(getattr(r, k), ref[k], err_msg=k)
        gd, gdt = api.diag_via_sum_diff(img, p)
        np.testing.assert_array_equal(gd, ref["gd"])
        np.testing.assert_array_equal(gdt, ref["gdt"])
    with pytest.raises(api.ImageTooSmall):
        api.sobel5_4d(np.zeros((4, 9), np.uint8))
