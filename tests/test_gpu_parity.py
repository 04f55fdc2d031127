"""GPU parity: the sm_100a kernels through the C ABI vs the oracle and the
reference's golden fixtures.  Integer planes and the clamp_abs uint8 map
must be bit-exact; the double magnitude is bit-exact too (the kernel
reproduces the reference's rounding sequence); the optional float magnitude
is within 1 ulp of the double one (tolerance stated in
test_float_magnitude_within_one_ulp)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PLANES = ("gx", "gy", "gd", "gdt", "g")
ALL = PLANES + ("g32", "u8")

with open(os.path.join(GOLD, "cases.json")) as f:
    CASES = json.load(f)
ARRS = np.load(os.path.join(GOLD, "cases.npz"))
with open(os.path.join(GOLD, "hashes.json")) as f:
    HASHES = json.load(f)


@pytest.fixture(scope="module")
def S(cuda):
    import paper_2305_00515_b200 as S
    return S


def run_device(S, img, taps, prefetch, planes=ALL):
    import torch
    from paper_2305_00515_b200 import api
    h, w = img.shape
    d_in, pitch = api.alloc_input(w, h)
    d_in.zero_()
    d_in[:, :w].copy_(torch.from_numpy(np.ascontiguousarray(img)))
    out, op = api.alloc_planes(w - 4, h - 4, planes)
    for v in out.values():
        v.fill_(0x5A if v.dtype == torch.uint8 else 7)  # poison: every pixel must be written
    diag = torch.zeros(8, dtype=torch.int32, device="cuda")
    api.launch(d_in, pitch, w, h, taps, prefetch, out, op, diag)
    torch.cuda.synchronize()
    return {k: v[:, : w - 4].cpu().numpy() for k, v in out.items()}, diag.cpu().tolist()


def taps_of(S, d):
    return S.Taps.from_dict(d)


@pytest.mark.parametrize("prefetch", [0, 1])
@pytest.mark.parametrize("i", range(len(CASES)), ids=[c["name"] for c in CASES])
def test_golden_case_device(S, i, prefetch):
    c = CASES[i]
    img = ARRS[f"img{i}"]
    taps = taps_of(S, c["taps"])
    if c["status"] == 13:
        with pytest.raises(S.ImageTooSmall):
            run_device(S, img, taps, prefetch)
        return
    got, diag = run_device(S, img, taps, prefetch)
    if c["status"] == 17:
        assert diag[0] > 0  # recover_diag parity violation recorded
        return
    assert diag[0] == 0
    for k in PLANES:
        np.testing.assert_array_equal(got[k], ARRS[f"{k}{i}"], err_msg=k)
    np.testing.assert_array_equal(got["u8"], ARRS[f"u8{i}"])


@pytest.mark.parametrize("i", range(len(CASES)), ids=[c["name"] for c in CASES])
def test_golden_case_run_stream_api(S, i):
    """The drop-in run_stream (host buffers, chunked copy pipeline)."""
    c = CASES[i]
    img = ARRS[f"img{i}"]
    w = img.shape[1]
    taps = taps_of(S, c["taps"])
    plan = S.plan_strips(max(w, 5), c["lanes"], 2)
    if c["status"] == 13:
        with pytest.raises(S.ImageTooSmall):
            S.run_stream(img, taps, plan, S.Prefetch.on)
        return
    if c["status"] == 17:
        with pytest.raises(S.ParityViolation) as ei:
            S.run_stream(img, taps, plan, S.Prefetch(c["prefetch"]))
        # the pair the reference reports (workers = 1: first in strip order)
        assert str(ei.value) == c["message"]
        return
    r = S.run_stream(img, taps, plan, S.Prefetch(c["prefetch"]))
    for k in PLANES:
        np.testing.assert_array_equal(getattr(r, k), ARRS[f"{k}{i}"], err_msg=k)
    assert r.counters == c["counters"]


def test_random_sweep_vs_oracle(S, oracle):
    """SPEC ACCEPTANCE 1 analogue: seeded random images 5x5..700x150, both
    kernel variants, default / non-default / fault-injected taps."""
    import pyoracle
    rng = np.random.default_rng(11)
    variants = [oracle.make_stream_taps(), oracle.make_stream_taps(2, 3, 5, 1),
                oracle.make_stream_taps(1, 32768, 1, 1)]
    fault = oracle.make_stream_taps()
    fault.k0[0] += 2
    variants.append(fault)
    for trial in range(48):
        w, h = int(rng.integers(5, 700)), int(rng.integers(5, 150))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        if trial % 3 == 0:
            img &= 7
        t = variants[trial % len(variants)]
        st, ref, _ = oracle.run_stream(img, t)
        assert st == 0
        got, diag = run_device(S, img, S.Taps.from_dict(t.as_dict()), trial % 2)
        assert diag[0] == 0
        for k in PLANES:
            np.testing.assert_array_equal(got[k], ref[k], err_msg=f"{k} {w}x{h} taps{trial % 4}")
        np.testing.assert_array_equal(got["u8"], oracle.clamp_abs(ref["g"]))
    del pyoracle


def test_float_magnitude_within_one_ulp(S, oracle):
    """g32: tolerance 1 ulp of float32 relative to the double magnitude."""
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (130, 777), dtype=np.uint8)
    got, _ = run_device(S, img, S.make_stream_taps(), 1)
    ref = got["g"]
    exact = ref.astype(np.float32)
    ulps = np.abs(got["g32"].view(np.int32).astype(np.int64) - exact.view(np.int32))
    assert ulps.max() <= 1


def test_subset_of_planes(S, oracle):
    """Only requested planes are written (NULL planes skipped)."""
    rng = np.random.default_rng(2)
    img = rng.integers(0, 256, (40, 300), dtype=np.uint8)
    st, ref, _ = oracle.run_stream(img)
    for planes in (("gx",), ("u8",), ("gd", "g"), ("gdt", "g32")):
        got, _ = run_device(S, img, S.make_stream_taps(), 1, planes)
        assert set(got) == set(planes)
        for k in planes:
            if k in ref:
                np.testing.assert_array_equal(got[k], ref[k])
        if "u8" in planes:
            np.testing.assert_array_equal(got["u8"], oracle.clamp_abs(ref["g"]))


def test_batch_launch(S, oracle):
    import torch
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(3)
    w, h, n = 301, 37, 5
    imgs = rng.integers(0, 256, (n, h, w), dtype=np.uint8)
    d_in, pitch = api.alloc_input(w, h, frames=n)
    d_in[:, :, :w].copy_(torch.from_numpy(imgs))
    out, op = api.alloc_planes(w - 4, h - 4, PLANES, frames=n)
    api.launch_batch(d_in, pitch, h * pitch, w, h, n, S.make_stream_taps(), 1, out, op,
                     (h - 4) * op)
    torch.cuda.synchronize()
    for f in range(n):
        st, ref, _ = oracle.run_stream(imgs[f])
        for k in PLANES:
            np.testing.assert_array_equal(out[k][f, :, : w - 4].cpu().numpy(), ref[k])


@pytest.mark.parametrize("n_bands,band", [(2, ""), (3, ""), (5, ""), (2, "4"), (3, "6"),
                                          (2, "8"), (3, "16")])
def test_row_band_partition_equals_whole(S, oracle, monkeypatch, n_bands, band):
    """C5 row-band tiler: bands with 2-row halos above/below stitch to the
    single-image result (the multi-GPU partition, exercised on one GPU).
    Forced CTA bands switch on the TMA rows (kGeomSegTma): CTAs whose rows
    touch a halo load from global memory, the others from shared memory."""
    import torch
    from paper_2305_00515_b200 import api
    if band:
        monkeypatch.setenv("SOBEL5_BAND", band)
    rng = np.random.default_rng(4)
    w, h = (1543, 157) if band else (523, 97)
    img = rng.integers(0, 256, (h, w), dtype=np.uint8)
    st, ref, _ = oracle.run_stream(img)
    bounds = np.linspace(0, h, n_bands + 1).astype(int)
    for b in range(n_bands):
        r0, r1 = int(bounds[b]), int(bounds[b + 1])
        body, pitch = api.alloc_input(w, r1 - r0)
        body[:, :w].copy_(torch.from_numpy(img[r0:r1]))
        top = bot = None
        if r0 > 0:
            top, _ = api.alloc_input(w, 2)
            top[:, :w].copy_(torch.from_numpy(img[r0 - 2:r0]))
        if r1 < h:
            bot, _ = api.alloc_input(w, 2)
            bot[:, :w].copy_(torch.from_numpy(img[r1:r1 + 2]))
        rows = (r1 - r0) + (2 if top is not None else 0) + (2 if bot is not None else 0) - 4
        out, op = api.alloc_planes(w - 4, rows, PLANES)
        api.launch_band(top, body, bot, pitch, w, r1 - r0, S.make_stream_taps(), 1, out, op)
        torch.cuda.synchronize()
        y0 = r0 - 2 if top is not None else 0
        for k in PLANES:
            np.testing.assert_array_equal(out[k][:, : w - 4].cpu().numpy(), ref[k][y0:y0 + rows],
                                          err_msg=f"band {b} {k}")


def test_device_synth_matches_reference_generator(S, oracle):
    import torch
    from paper_2305_00515_b200 import api
    for (w, h, seed, mask) in [(16, 1, 1, 0xFF), (1920, 1080, 1, 0xFF), (333, 17, 9, 0x07)]:
        d, pitch = api.alloc_input(w, h)
        api.synth_random_device(d, pitch, w, h, seed, mask)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(d[:, :w].cpu().numpy(),
                                      oracle.synth_random(w, h, seed) & mask)
    # a band generated with a row offset equals the same rows of the full image
    d, pitch = api.alloc_input(100, 7)
    api.synth_random_device(d, pitch, 100, 7, 5, 0xFF, row_offset=13)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(d[:, :100].cpu().numpy(),
                                  oracle.synth_random(100, 20, 5)[13:20])


@pytest.mark.parametrize("key", list(HASHES))
def test_golden_hashes_full_size(S, oracle, key):
    """Full-size C1..C3 planes hashed against the reference's FNV-1a values."""
    import torch
    from paper_2305_00515_b200 import api
    e = HASHES[key]
    w, h = e["w"], e["h"]
    d_in, pitch = api.alloc_input(w, h)
    api.synth_random_device(d_in, pitch, w, h, e["seed"], e["mask"])
    out, op = api.alloc_planes(w - 4, h - 4, PLANES + ("u8",))
    diag = torch.zeros(8, dtype=torch.int32, device="cuda")
    api.launch(d_in, pitch, w, h, S.make_stream_taps(), 1, out, op, diag)
    torch.cuda.synchronize()
    assert diag[0].item() == 0
    assert f"{oracle.fnv1a64(d_in[:, :w].cpu().numpy()):016x}" == e["fnv1a64"]["input"]
    for k in PLANES + ("u8",):
        host = np.ascontiguousarray(out[k][:, : w - 4].cpu().numpy())
        assert f"{oracle.fnv1a64(host):016x}" == e["fnv1a64"][k], k


def test_launch_count_increments(S):
    from paper_2305_00515_b200 import api
    before = api.launch_count()
    run_device(S, np.zeros((8, 8), np.uint8), S.make_stream_taps(), 1)
    assert api.launch_count() == before + 1


def test_misaligned_arguments_rejected(S):
    import torch
    from paper_2305_00515_b200 import api
    d_in, pitch = api.alloc_input(64, 16)
    out, op = api.alloc_planes(60, 12, ("gx",))
    with pytest.raises(S.Error):  # pitch not a multiple of 16
        api.launch(d_in, 65, 64, 16, S.make_stream_taps(), 1, out, op)
    with pytest.raises(S.Error):  # output pitch below width-4
        api.launch(d_in, pitch, 64, 16, S.make_stream_taps(), 1, out, 56)
    del torch


@pytest.mark.parametrize("which,hi", [(0, 1 << 30), (1, 1 << 31), (2, 65281), (3, 0x7F800000),
                                      (4, 65281), (5, 0x7F800000)],
                         ids=["sqrt_u30", "u8_from_s", "u8_float_exact", "u8_float_saturated",
                              "u8_sqrt_exact", "u8_sqrt_saturated"])
def test_epilogue_arithmetic_exhaustive(S, which, hi):
    """The fast epilogue is bit-identical to IEEE sqrt (which=0) and to
    clamp_abs(round(sqrt)) (which=1) for EVERY integer sum of squares the
    packed kernel can produce (default taps: S <= 4 * 12240^2 < 2^30); the
    u8-only kernels' packed-float epilogue is exact for every integer S <=
    65280 (which=2) and saturates for every float S >= 65281 (which=3); the
    same for the u8-only kernel's sqrt + saturating round (which=4/5,
    sobel5_u8.cuh)."""
    import torch
    from paper_2305_00515_b200 import _abi
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    S.api.check(_abi.load().sobel5_selftest(which, 0, hi, cnt.data_ptr(), None), "selftest")
    torch.cuda.synchronize()
    assert cnt.item() == 0


@pytest.mark.parametrize("extra", [0, 4, 12])
def test_plane_pitch_variants(S, oracle, extra):
    """Output pitch = round_up(out_w, 4) + extra elements: the lane-pair
    256-bit stores need 8-column (32-B) aligned rows and fall back to 128-bit
    stores otherwise; both must write exactly the valid columns."""
    import torch
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(extra + 1)
    for w, h in ((301, 37), (1029, 21), (517, 9)):
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        d_in, pitch = api.alloc_input(w, h)
        d_in[:, :w].copy_(torch.from_numpy(img))
        ow, oh = w - 4, h - 4
        op = (ow + 3) // 4 * 4 + extra
        dt = {"gx": torch.int32, "gy": torch.int32, "gd": torch.int32, "gdt": torch.int32,
              "g": torch.float64}
        out = {}
        for k in PLANES:  # 32-B aligned bases, poisoned
            t = torch.full((oh * op + 8,), 7, dtype=dt[k], device="cuda")
            off = (-(t.data_ptr() // t.element_size())) % (32 // t.element_size())
            out[k] = t[off:off + oh * op].view(oh, op)
        api.launch(d_in, pitch, w, h, S.make_stream_taps(), 1, out, op)
        torch.cuda.synchronize()
        st, ref, _ = oracle.run_stream(img)
        for k in PLANES:
            got = out[k].cpu().numpy()
            np.testing.assert_array_equal(got[:, :ow], ref[k], err_msg=f"{k} pitch {op}")
            if op > ow:
                assert (got[:, ow:] == 7).all(), f"{k}: wrote past the row (pitch {op})"


def test_ablation_kernels_bit_exact(S, oracle, monkeypatch):
    """The dense-correlation ablation kernel (SOBEL5_DENSE=1, no operator
    transformation) gives the same planes and u8 map as the oracle."""
    monkeypatch.setenv("SOBEL5_DENSE", "1")
    rng = np.random.default_rng(17)
    for w, h, mask in ((517, 61, 0xFF), (130, 33, 0x07), (5, 5, 0xFF)):
        img = (rng.integers(0, 256, (h, w), dtype=np.uint8) & mask).astype(np.uint8)
        st, ref, _ = oracle.run_stream(img)
        got, _ = run_device(S, img, S.make_stream_taps(), 1, PLANES)
        for k in PLANES:
            np.testing.assert_array_equal(got[k], ref[k], err_msg=k)
        got, _ = run_device(S, img, S.make_stream_taps(), 1, ("u8",))
        np.testing.assert_array_equal(got["u8"], oracle.clamp_abs(ref["g"]))


@pytest.mark.parametrize("band", ["8", "16", "32"])
def test_tma_band_loads_any_band(S, oracle, monkeypatch, band):
    """TMA band loads (kGeomPlainTma) with forced bands up to the 36-row
    shared-memory limit: more band rows than warp-0 lanes must all be issued
    (bulk copies loop over the rows), ragged last band, batch frames."""
    import torch
    from paper_2305_00515_b200 import api
    monkeypatch.setenv("SOBEL5_BAND", band)
    rng = np.random.default_rng(int(band))
    for w, h, n in ((1541, 77, 1), (600, 45, 3)):
        imgs = rng.integers(0, 256, (n, h, w), dtype=np.uint8)
        d_in, pitch = api.alloc_input(w, h, frames=n)
        d_in.view(n, h, pitch)[:, :, :w].copy_(torch.from_numpy(imgs))
        out, op = api.alloc_planes(w - 4, h - 4, PLANES, frames=n)
        if n > 1:
            api.launch_batch(d_in, pitch, h * pitch, w, h, n, S.make_stream_taps(), 1, out, op,
                             (h - 4) * op)
        else:
            api.launch(d_in, pitch, w, h, S.make_stream_taps(), 1, out, op)
        torch.cuda.synchronize()
        for f in range(n):
            st, ref, _ = oracle.run_stream(imgs[f])
            for k in PLANES:
                got = out[k].view(n, h - 4, op)[f, :, : w - 4].cpu().numpy()
                np.testing.assert_array_equal(got, ref[k], err_msg=f"band {band} {k} frame {f}")


@pytest.mark.parametrize("lanes", [8, 37, 64, 4096])
@pytest.mark.parametrize("kind", ["packed_runtime_taps", "f32x2_runtime_taps", "generic"])
def test_parity_violation_pair_matches_reference(reference, lanes, kind):
    """Fault-injected taps with odd pairs in many strips and rows: the pair
    every GPU kernel family reports is the one the compiled reference's
    run_stream raises with workers = 1 (first odd pixel in strip, row,
    column order; sobel5_diag, pipeline.hpp:416-445 / 268-273)."""
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(lanes)
    h, w = 97, 301
    img = rng.integers(0, 256, (h, w), dtype=np.uint8)
    params = {"packed_runtime_taps": (1, 1, 1, 1), "f32x2_runtime_taps": (2, 3, 5, 7),
              "generic": (1, 32768, 1, 1)}[kind]
    code, t, msg = reference.make_stream_taps(*params)
    assert code == 0, msg
    t.k1[2] += 1  # odd fault: P + M odd wherever the centre pixel is odd
    taps = api.Taps.from_dict(t.as_dict())
    assert api.kernel_for(taps) == kind
    code, _, _, want = reference.run_stream(img, t, lanes=lanes, prefetch=True, workers=1)
    assert code == 17 and want.startswith("odd sum/difference pair ("), (code, want)
    plan = api.plan_strips(w, lanes, 2)
    with pytest.raises(api.ParityViolation) as ei:
        api.run_stream(img, taps, plan, api.Prefetch.on)
    assert str(ei.value) == want


def _fault_taps(reference):
    from paper_2305_00515_b200 import api
    code, t, msg = reference.make_stream_taps(1, 1, 1, 1)
    assert code == 0, msg
    t.k1[2] += 1  # odd P + M wherever the centre pixels of rows v+1, v+3 differ in parity
    return t, api.Taps.from_dict(t.as_dict())


def _noisy(img, rng, rows, cols):
    """Random pixels in input rows [r0, r1) x columns [c0, c1) of a flat image
    (a flat region has no odd pairs under the fault)."""
    (r0, r1), (c0, c1) = rows, cols
    img[r0:r1, c0:c1] = rng.integers(0, 256, (r1 - r0, c1 - c0), dtype=np.uint8)


@pytest.mark.parametrize("layout", ["same_strip", "later_strip"])
def test_parity_pair_across_row_chunks(reference, layout):
    """sobel5_run_host cuts a tall image into row chunks (>= 256 output rows
    each, one launch per chunk); the order key of a pair is global, so the
    reported pair is the reference's first in (strip, row, column) order even
    when a later chunk holds odd pixels at smaller chunk-local rows."""
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(5)
    h, w, lanes = 900, 301, 64  # strips of 60 output columns; chunks 0..255, 256..511, ...
    img = np.zeros((h, w), np.uint8)
    a_cols = (10, 40) if layout == "same_strip" else (130, 160)  # strip 0 or strip 2
    _noisy(img, rng, (200, 216), a_cols)   # chunk 0, rows ~196..215
    _noisy(img, rng, (300, 311), (5, 50))  # chunk 1 (local rows ~40..54), strip 0
    t, taps = _fault_taps(reference)
    code, _, _, want = reference.run_stream(img, t, lanes=lanes, prefetch=True, workers=1)
    assert code == 17, want
    with pytest.raises(api.ParityViolation) as ei:
        api.run_stream(img, taps, api.plan_strips(w, lanes, 2), api.Prefetch.on)
    assert str(ei.value) == want


@pytest.mark.parametrize("transport", ["peer", "copy"])
def test_parity_pair_across_bands(reference, transport):
    """The multi-GPU row bands (device list {0, 0, 0}): band keys are global
    rows and the merge keeps the earliest, so the pair is the reference's even
    when a later band has an odd pixel at a smaller band-local row."""
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(9)
    h, w, lanes = 300, 301, 64
    img = np.zeros((h, w), np.uint8)
    _noisy(img, rng, (20, 31), (130, 160))   # band 0, strip 2
    _noisy(img, rng, (150, 161), (5, 50))    # band 1, strip 0, band-local rows ~46..
    _noisy(img, rng, (205, 211), (5, 50))    # band 2, strip 0, band-local rows ~1..
    t, taps = _fault_taps(reference)
    code, _, _, want = reference.run_stream(img, t, lanes=lanes, prefetch=True, workers=1)
    assert code == 17, want
    with pytest.raises(api.ParityViolation) as ei:
        api.run_stream_bands(img, taps, api.plan_strips(w, lanes, 2), api.Prefetch.on, [0, 0, 0],
                             transport)
    assert str(ei.value) == want
