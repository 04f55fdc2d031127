"""GPU: the int16 D2H wire of the host path (sobel5_ctx.cu, sobel5_wire.cpp).

With default taps and exactly the StreamResult planes, sobel5_run_host ships
gx, gy, gd, gdt over PCIe as int16 (every packed-kernel gradient lies in
[-2^15, 2^15)) and widens them into the caller's int32 planes; the split
begin/_staging form exposes the int16 staging (sobel5_run_host_staging_elem
== 2).  The magnitude g does not cross PCIe on the chunk-major wire: the host
rebuilds it from the int16 rows (wire "1"); SOBEL5_WIRE_G=0 ships it as f64
(wire "g0").  Whatever the wire, the planes must equal the oracle's run_stream
(pipeline.hpp:452-477) bit for bit, including the extreme gradients."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PLANES = ("gx", "gy", "gd", "gdt", "g")
DT = {"gx": np.int32, "gy": np.int32, "gd": np.int32, "gdt": np.int32, "g": np.float64}


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


def extreme_image(h, w):
    """8-pixel stripes of 0 / 255, vertical (top third: gx = +-12240, the
    maximum of the (1,2,6,4) taps), horizontal (middle: gy = +-12240) and an
    8x8 checkerboard (bottom: the diagonal responses)."""
    y, x = np.mgrid[0:h, 0:w]
    img = (((x // 8) + (y // 8)) % 2 * 255).astype(np.uint8)
    img[: h // 3] = ((x[: h // 3] // 8) % 2 * 255).astype(np.uint8)
    img[h // 3: 2 * h // 3] = ((y[h // 3: 2 * h // 3] // 8) % 2 * 255).astype(np.uint8)
    return img


@pytest.mark.parametrize("wire", ["1", "g0", "0"])
@pytest.mark.parametrize("h,w,kind", [(5, 5, "rand"), (6, 9, "rand"), (300, 5, "rand"),
                                      (61, 97, "rand"), (300, 1031, "extreme"),
                                      (4400, 1027, "rand"), (2100, 4099, "extreme")])
def test_run_host_sr_wire(ctx, oracle, monkeypatch, wire, h, w, kind):
    import torch
    from paper_2305_00515_b200 import _abi, api
    monkeypatch.setenv("SOBEL5_WIRE16", "0" if wire == "0" else "1")
    monkeypatch.setenv("SOBEL5_WIRE_G", "0" if wire == "g0" else "1")
    img = (np.random.default_rng(h * w).integers(0, 256, (h, w), dtype=np.uint8)
           if kind == "rand" else extreme_image(h, w))
    st, ref, _ = oracle.run_stream(img)
    assert st == 0
    if kind == "extreme":
        for k in ("gx", "gy"):
            assert int(ref[k].max()) == 12240 and int(ref[k].min()) == -12240, k
    ow, oh = w - 4, h - 4
    taps = api.make_stream_taps()
    L = _abi.load()
    d = _abi.Diag()
    # pageable planes (odd widths: rows start at every alignment)
    res = {k: np.full((oh, ow), 7, DT[k]) for k in PLANES}
    assert L.sobel5_run_host(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1,
                             C.byref(planes_struct(res, ow)), C.byref(d)) == 0
    for k in PLANES:
        np.testing.assert_array_equal(res[k], ref[k], err_msg=f"pageable {k} wire={wire}")
    # bytes over PCIe: the four int16 planes as one block per row chunk (rows
    # padded to 32 elements) (+ f64 g with SOBEL5_WIRE_G=0), 4 x int32 + f64
    # without the wire
    dp = (ow + 31) // 32 * 32
    want = {"1": 4 * dp * oh * 2, "g0": 4 * dp * oh * 2 + ow * oh * 8, "0": ow * oh * 24}[wire]
    assert L.sobel5_ctx_last_d2h_bytes(ctx.handle) == want
    # page-locked planes (the bench's e2e path)
    pin = {k: torch.full((oh, ow), 7, dtype=getattr(torch, np.dtype(DT[k]).name)).pin_memory()
           for k in PLANES}
    h_in = torch.from_numpy(img).pin_memory()
    assert L.sobel5_run_host(ctx.handle, h_in.data_ptr(), w, h, C.byref(taps), 1,
                             C.byref(planes_struct(pin, ow)), C.byref(d)) == 0
    for k in PLANES:
        np.testing.assert_array_equal(pin[k].numpy(), ref[k], err_msg=f"pinned {k} wire={wire}")


@pytest.mark.parametrize("wire", ["2", "1", "0"])
def test_staging_elem_and_consumer(ctx, oracle, monkeypatch, wire):
    """begin(0x1f) -> _staging_elem / _staging (int16 unless SOBEL5_WIRE16=0)
    -> the consumer widens the rows itself -> finish(NULL)."""
    from paper_2305_00515_b200 import _abi, api
    monkeypatch.setenv("SOBEL5_WIRE16", wire)
    L = _abi.load()
    h, w = 2300, 517
    img = extreme_image(h, w)
    st, ref, _ = oracle.run_stream(img)
    ow, oh = w - 4, h - 4
    taps = api.make_stream_taps()
    assert L.sobel5_run_host_staging_elem(ctx.handle, 0) == 0  # nothing pending
    assert L.sobel5_run_host_begin(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1, 0x1F) == 0
    want = 2 if wire in ("1", "2") else 4
    assert [L.sobel5_run_host_staging_elem(ctx.handle, i) for i in range(7)] == \
        [want] * 4 + [8, 0, 0]
    y0, y1, k = C.c_int(), C.c_int(), 0
    while L.sobel5_run_host_chunk(ctx.handle, k, C.byref(y0), C.byref(y1)) == 0:
        k += 1
    assert y1.value == oh
    for i, name in enumerate(PLANES):
        es = L.sobel5_run_host_staging_elem(ctx.handle, i)
        dt = {2: np.int16, 4: np.int32, 8: np.float64}[es]
        buf = (C.c_char * (ow * oh * es)).from_address(L.sobel5_run_host_staging(ctx.handle, i))
        arr = np.frombuffer(buf, dtype=dt).reshape(oh, ow).astype(DT[name])
        np.testing.assert_array_equal(arr, ref[name], err_msg=name)
    d = _abi.Diag()
    assert L.sobel5_run_host_finish(ctx.handle, None, C.byref(d)) == 0


def test_wire_not_for_custom_taps_or_other_masks(ctx, oracle):
    """Taps other than the default ones, or a mask other than 0x1f, keep the
    int32 wire (the int16 bound is proven for the default taps only)."""
    from paper_2305_00515_b200 import _abi, api
    L = _abi.load()
    h, w = 300, 203
    img = np.random.default_rng(5).integers(0, 256, (h, w), dtype=np.uint8)
    taps = api.make_stream_taps(api.FilterParams(1, 1, 1, 1))
    assert L.sobel5_run_host_begin(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1, 0x1F) == 0
    assert L.sobel5_run_host_staging_elem(ctx.handle, 0) == 4
    st, ref, _ = oracle.run_stream(img, oracle.make_stream_taps(1, 1, 1, 1))
    res = {k: np.zeros((h - 4, w - 4), DT[k]) for k in PLANES}
    d = _abi.Diag()
    assert L.sobel5_run_host_finish(ctx.handle, C.byref(planes_struct(res, w - 4)), C.byref(d)) == 0
    for k in PLANES:
        np.testing.assert_array_equal(res[k], ref[k], err_msg=k)
    dflt = api.make_stream_taps()
    assert L.sobel5_run_host_begin(ctx.handle, img.ctypes.data, w, h, C.byref(dflt), 1, 0x0F) == 0
    assert L.sobel5_run_host_staging_elem(ctx.handle, 0) == 4
    assert L.sobel5_run_host_finish(ctx.handle, None, C.byref(d)) == 0


def test_split_form_finish_widens(ctx, oracle, monkeypatch):
    """begin(0x1f) -> finish(h_out) widens the int16 staging into the
    caller's int32 planes (several row chunks)."""
    from paper_2305_00515_b200 import _abi, api
    monkeypatch.setenv("SOBEL5_WIRE16", "2")
    L = _abi.load()
    h, w = 3000, 771
    img = extreme_image(h, w)
    st, ref, _ = oracle.run_stream(img)
    taps = api.make_stream_taps()
    assert L.sobel5_run_host_begin(ctx.handle, img.ctypes.data, w, h, C.byref(taps), 1, 0x1F) == 0
    assert L.sobel5_run_host_staging_elem(ctx.handle, 3) == 2
    res = {k: np.full((h - 4, w - 4), 7, DT[k]) for k in PLANES}
    d = _abi.Diag()
    assert L.sobel5_run_host_finish(ctx.handle, C.byref(planes_struct(res, w - 4)), C.byref(d)) == 0
    for k in PLANES:
        np.testing.assert_array_equal(res[k], ref[k], err_msg=k)


@pytest.mark.parametrize("wire", ["1", "g0", "0"])
@pytest.mark.parametrize("h,w", [(3, 3), (61, 97), (2300, 1027), (700, 4099)])
def test_sobel3_run_host_wire(ctx, oracle, monkeypatch, wire, h, w):
    """run_stream_3x3's host path: gx, gy over the int16 wire (|gx|, |gy| <=
    1020), widened into the caller's int32 planes; g rebuilt on the host (or
    as f64 with SOBEL5_WIRE_G=0)."""
    import torch
    from paper_2305_00515_b200 import _abi
    monkeypatch.setenv("SOBEL5_WIRE16", "0" if wire == "0" else "1")
    monkeypatch.setenv("SOBEL5_WIRE_G", "0" if wire == "g0" else "1")
    L = _abi.load()
    img = np.random.default_rng(h + 7 * w).integers(0, 256, (h, w), dtype=np.uint8)
    if h > 100:
        img[: h // 2] = extreme_image(h // 2, w)[:, :w]
    st, ref = oracle.sobel3_2d(img)
    assert st == 0
    ow, oh = w - 2, h - 2
    for pinned in (False, True):
        res = {k: np.full((oh, ow), 7, DT[k]) for k in ("gx", "gy", "g")}
        if pinned:
            res = {k: torch.from_numpy(v).pin_memory() for k, v in res.items()}
        assert L.sobel3_run_host(ctx.handle, img.ctypes.data, w, h, 1,
                                 C.byref(planes_struct(res, ow))) == 0
        for k in ("gx", "gy", "g"):
            got = res[k].numpy() if pinned else res[k]
            np.testing.assert_array_equal(got, ref[k], err_msg=f"{k} pinned={pinned} wire={wire}")
        dp = (ow + 31) // 32 * 32
        want = {"1": 2 * dp * oh * 2, "g0": 2 * dp * oh * 2 + ow * oh * 8, "0": ow * oh * 16}[wire]
        assert L.sobel5_ctx_last_d2h_bytes(ctx.handle) == want
