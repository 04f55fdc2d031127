"""GPU parity of the detect path through the C ABI:
fused replicate padding (pad_replicate, image_io.hpp:279-291) and the u8
export of g in both SaveModes (detail::quantize, image_io.hpp:233-256),
against the C oracle (itself pinned to the compiled reference in
tests/test_detect_oracle.py and tests/golden/detect.npz).  Everything is
bit-exact: integer planes, the double magnitude and both u8 maps."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SR = ("gx", "gy", "gd", "gdt", "g")
DT = {"gx": np.int32, "gy": np.int32, "gd": np.int32, "gdt": np.int32, "g": np.float64}

# widths around the lane (4 px), warp (128) and CTA (512) tiles, both edges
SIZES = [(1, 1), (1, 7), (7, 1), (2, 3), (5, 5), (61, 97), (17, 127), (9, 128), (9, 129),
         (6, 130), (13, 131), (4, 132), (33, 255), (3, 256), (21, 509), (7, 512), (11, 513),
         (5, 645), (70, 40), (300, 260)]


@pytest.fixture(scope="module")
def api(cuda):
    from paper_2305_00515_b200 import api
    return api


def to_dev(api, img, frames=None):
    import torch
    if img.ndim == 2:
        h, w = img.shape
        d, pitch = api.alloc_input(w, h)
        d.fill_(0xA5)  # poison beyond the width: the kernel must not read it as pixels
        d[:, :w].copy_(torch.from_numpy(np.ascontiguousarray(img)))
    else:
        n, h, w = img.shape
        d, pitch = api.alloc_input(w, h, frames=n)
        d.fill_(0xA5)
        d[:, :, :w].copy_(torch.from_numpy(np.ascontiguousarray(img)))
    return d, pitch


def padded_ref(oracle, img, taps=None):
    st, padded = oracle.pad_replicate(img, 2)
    assert st == 0
    st, ref, _ = oracle.run_stream(padded, taps)
    assert st == 0
    return ref


def rand_img(h, w, seed, mask=0xFF):
    return (np.random.default_rng(seed).integers(0, 256, (h, w), dtype=np.uint8) & mask).astype(
        np.uint8)


@pytest.mark.parametrize("prefetch", [0, 1])
@pytest.mark.parametrize("h,w", SIZES)
def test_pad_launch_all_planes(api, oracle, h, w, prefetch):
    import torch
    img = rand_img(h, w, h * 1000 + w, 0x07 if (h + w) % 2 else 0xFF)
    d, pitch = to_dev(api, img)
    out, op = api.alloc_planes(w, h, SR + ("u8",))
    for v in out.values():
        v.fill_(7)
    api.launch_ex(d, pitch, w, h, api.make_stream_taps(), prefetch, True, out, op)
    torch.cuda.synchronize()
    ref = padded_ref(oracle, img)
    for k in SR:
        np.testing.assert_array_equal(out[k][:, :w].cpu().numpy(), ref[k], err_msg=k)
    np.testing.assert_array_equal(out["u8"][:, :w].cpu().numpy(), oracle.clamp_abs(ref["g"]))


@pytest.mark.parametrize("params", [(1, 1, 1, 1), (2, 3, 5, 7), (1, 32768, 1, 1)])
@pytest.mark.parametrize("h,w", [(1, 1), (9, 129), (40, 515), (23, 37)])
def test_pad_generic_taps(api, oracle, h, w, params):
    """Non-default taps take the generic kernel, also with fused padding."""
    import torch
    sys_taps = oracle.make_stream_taps(*params)
    taps = api.Taps.from_dict(sys_taps.as_dict())
    img = rand_img(h, w, 7 + h + w)
    d, pitch = to_dev(api, img)
    out, op = api.alloc_planes(w, h, SR)
    api.launch_ex(d, pitch, w, h, taps, 1, True, out, op)
    torch.cuda.synchronize()
    ref = padded_ref(oracle, img, sys_taps)
    for k in SR:
        np.testing.assert_array_equal(out[k][:, :w].cpu().numpy(), ref[k], err_msg=k)


def _detect(api, img, pad, mode, planes=(), taps=None, prefetch=1):
    import torch
    h, w = img.shape
    ow, oh = (w, h) if pad else (w - 4, h - 4)
    d, pitch = to_dev(api, img)
    out, op = api.alloc_planes(ow, oh, tuple(planes) + ("u8",))
    out["u8"].fill_(0x5A)
    scratch = api.alloc_scratch(1, out_h=oh, pitch=op)
    api.detect_device(d, pitch, w, h, taps or api.make_stream_taps(), prefetch, pad, mode, out,
                      op, scratch)
    torch.cuda.synchronize()
    return {k: v[:, :ow].cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("mode", ["clamp_abs", "normalize"])
@pytest.mark.parametrize("pad", [True, False])
@pytest.mark.parametrize("h,w,mask", [(61, 97, 0xFF), (61, 97, 0x07), (5, 5, 0xFF), (1, 1, 0xFF),
                                      (130, 517, 0x03), (33, 129, 0x01), (8, 600, 0x3F)])
def test_detect_modes(api, oracle, h, w, mask, pad, mode):
    if not pad and (h < 5 or w < 5):
        pytest.skip("valid mode needs 5x5")
    img = rand_img(h, w, 3 * h + w, mask)
    got = _detect(api, img, pad, api.SaveMode[mode], planes=("g",))
    ref = padded_ref(oracle, img) if pad else oracle.run_stream(img)[1]
    np.testing.assert_array_equal(got["g"], ref["g"])
    np.testing.assert_array_equal(got["u8"], oracle.quantize(ref["g"], mode))


@pytest.mark.parametrize("kind", ["constant", "impulse", "ramp", "step", "two_level"])
def test_detect_normalize_edge_cases(api, oracle, kind):
    """span 0 (constant -> all 0), tiny spans and ties of the affine map."""
    h, w = 40, 150
    img = np.zeros((h, w), np.uint8)
    if kind == "constant":
        img[:] = 77
    elif kind == "impulse":
        img[20, 75] = 1
    elif kind == "ramp":
        img[:] = (np.arange(w) % 256).astype(np.uint8)
    elif kind == "step":
        img[:, 70:] = 255
    else:
        img[:, ::2] = 1
    got = _detect(api, img, True, api.SaveMode.normalize, planes=("g",))
    ref = padded_ref(oracle, img)
    np.testing.assert_array_equal(got["g"], ref["g"])
    np.testing.assert_array_equal(got["u8"], oracle.quantize(ref["g"], "normalize"))


@pytest.mark.parametrize("one_step", ["1", "0"])
@pytest.mark.parametrize("kind", ["random", "low", "checker", "narrow_span", "texture_ramp"])
def test_normalize_map_forms(api, oracle, monkeypatch, kind, one_step):
    """The S-plane map in both forms -- one compare against thr[j] when the
    float estimate is within 1/4 step (hi * 255 / span <= 2^16), estimate +
    check + search otherwise (SOBEL5_NORM_ONE_STEP=0 forces it) -- on
    images whose g spans are wide, small and narrow (lo close to hi: the
    one-compare form is refused and the search decides)."""
    monkeypatch.setenv("SOBEL5_NORM_ONE_STEP", one_step)
    h, w = 203, 1031
    rng = np.random.default_rng(7)
    if kind == "random":
        img = rand_img(h, w, 5)
    elif kind == "low":
        img = rand_img(h, w, 6, 0x03)
    elif kind == "checker":
        yy, xx = np.mgrid[0:h, 0:w]
        img = np.where((yy + xx) % 2 == 0, 255, 0).astype(np.int32)
        img = np.clip(img + rng.integers(-1, 2, (h, w)), 0, 255).astype(np.uint8)
    elif kind == "narrow_span":
        # a steep vertical ramp (every valid-mode g = 1488.96) with one
        # corner pixel raised: g spans [1488.96, 1492.72], hi * 255 / span =
        # 1.0e5 > 2^16, so the table refuses the one-compare form (valid
        # mode; replicate padding widens the span again)
        img = (8 * np.mgrid[0:30, 0:w][0]).astype(np.uint8)
        img[0, 0] += 1
    else:
        img = ((np.arange(w)[None, :] * 3 + np.arange(h)[:, None] * 5) % 256).astype(np.uint8)
        img ^= rng.integers(0, 4, (h, w), dtype=np.uint8)
    for pad in (True, False):
        got = _detect(api, img, pad, api.SaveMode.normalize, planes=("g",))
        ref = padded_ref(oracle, img) if pad else oracle.run_stream(img)[1]
        np.testing.assert_array_equal(got["g"], ref["g"])
        np.testing.assert_array_equal(got["u8"], oracle.quantize(ref["g"], "normalize"),
                                      err_msg=f"{kind} pad={pad}")


def test_normalize_map_1080p(api, oracle):
    """A full 1080p frame through the one-compare map (2 M pixels against
    the oracle's quantize of the oracle's g)."""
    img = rand_img(1080, 1920, 42)
    got = _detect(api, img, True, api.SaveMode.normalize, planes=("g",))
    ref = padded_ref(oracle, img)
    np.testing.assert_array_equal(got["g"], ref["g"])
    np.testing.assert_array_equal(got["u8"], oracle.quantize(ref["g"], "normalize"))


def test_detect_normalize_generic_taps(api, oracle):
    """Non-default taps: the generic kernel maps g with the direct formula."""
    sys_taps = oracle.make_stream_taps(2, 3, 5, 7)
    taps = api.Taps.from_dict(sys_taps.as_dict())
    img = rand_img(50, 300, 11, 0x0F)
    got = _detect(api, img, True, api.SaveMode.normalize, planes=("g",), taps=taps)
    ref = padded_ref(oracle, img, sys_taps)
    np.testing.assert_array_equal(got["g"], ref["g"])
    np.testing.assert_array_equal(got["u8"], oracle.quantize(ref["g"], "normalize"))


def test_detect_batch_per_frame_normalize(api, oracle):
    """Batched frames normalize with their own min/max."""
    import torch
    n, h, w = 4, 37, 141
    frames = np.stack([rand_img(h, w, 100 + i, [0xFF, 0x07, 0x01, 0x3F][i]) for i in range(n)])
    d, pitch = to_dev(api, frames)
    out, op = api.alloc_planes(w, h, ("u8",), frames=n)
    scratch = api.alloc_scratch(n, out_h=h, pitch=op, out_frame_stride=h * op)
    api.detect_device(d, pitch, w, h, api.make_stream_taps(), 1, True, api.SaveMode.normalize,
                      out, op, scratch, frames=n, in_frame_stride=h * pitch,
                      out_frame_stride=h * op)
    torch.cuda.synchronize()
    for i in range(n):
        ref = padded_ref(oracle, frames[i])
        np.testing.assert_array_equal(out["u8"][i, :, :w].cpu().numpy(),
                                      oracle.quantize(ref["g"], "normalize"), err_msg=str(i))


@pytest.mark.parametrize("mode", ["clamp_abs", "normalize"])
@pytest.mark.parametrize("dtype", ["f64", "i32"])
def test_quantize_device_plane(api, oracle, mode, dtype):
    rng = np.random.default_rng(5)
    if dtype == "f64":
        plane = rng.normal(0, 300, (57, 91))
        plane[0, :3] = [0.5, 1.5, 254.5]  # clamp_abs ties round away from zero
    else:
        plane = rng.integers(-70000, 70000, (57, 91)).astype(np.int32)
        plane[0, :3] = [0, 1, 2]
    got = api.quantize(plane, api.SaveMode[mode])
    np.testing.assert_array_equal(got, oracle.quantize(plane, mode))


def test_quantize_normalize_ties(api, oracle):
    """(v - lo) * 255 / span hits k + 0.5 exactly: lround rounds away."""
    plane = np.array([[0, 1, 2, 1]], np.int32)
    got = api.quantize(plane, api.SaveMode.normalize)
    np.testing.assert_array_equal(got, oracle.quantize(plane, "normalize"))
    assert got.tolist() == [[0, 128, 255, 128]]
    const = np.full((3, 3), 9.0)
    assert api.quantize(const, api.SaveMode.normalize).tolist() == [[0] * 3] * 3


@pytest.mark.parametrize("pad", [True, False])
@pytest.mark.parametrize("mode", ["clamp_abs", "normalize"])
def test_detect_host_api(api, oracle, pad, mode):
    """The host-buffer detect (the CLI's detect command on the GPU)."""
    img = rand_img(77, 203, 9, 0x1F)
    u8, planes = api.detect(img, api.FilterParams(), pad=pad, save_mode=api.SaveMode[mode],
                            planes=("gx", "g"))
    ref = padded_ref(oracle, img) if pad else oracle.run_stream(img)[1]
    np.testing.assert_array_equal(planes["gx"], ref["gx"])
    np.testing.assert_array_equal(planes["g"], ref["g"])
    np.testing.assert_array_equal(u8, oracle.quantize(ref["g"], mode))
    if pad:  # the PaddedPlane form of the reference flow (pad_replicate then run)
        pp = api.pad_replicate(img, 2)
        np.testing.assert_array_equal(api.detect(pp, save_mode=api.SaveMode[mode]), u8)


def test_detect_errors(api):
    with pytest.raises(api.EmptyPlane):
        api.detect(np.zeros((0, 0), np.uint8))
    with pytest.raises(api.ImageTooSmall):
        api.detect(np.zeros((4, 9), np.uint8), pad=False)
    u8 = api.detect(np.full((1, 1), 200, np.uint8), save_mode=api.SaveMode.clamp_abs)
    assert u8.tolist() == [[0]]


def test_detect_golden_fixtures(api):
    """tests/golden/detect.npz, generated from the compiled reference
    (pad_replicate + run_stream + detail::quantize)."""
    path = os.path.join(GOLD, "detect.npz")
    z = np.load(path)
    names = sorted({k.split("__")[0] for k in z.files})
    assert names
    for n in names:
        img = z[f"{n}__img"]
        for mode in ("clamp_abs", "normalize"):
            u8 = api.detect(img, pad=True, save_mode=api.SaveMode[mode])
            np.testing.assert_array_equal(u8, z[f"{n}__{mode}"], err_msg=f"{n} {mode}")


@pytest.mark.parametrize("mode", ["clamp_abs", "normalize"])
def test_quantize_device_pitched(api, oracle, mode):
    """sobel5_quantize_plane on pitched device planes (the dump-planes path)."""
    import torch
    rng = np.random.default_rng(12)
    plane = rng.integers(-5000, 5000, (33, 70)).astype(np.int32)
    d = torch.zeros((33, 96), dtype=torch.int32, device="cuda")
    d[:, :70] = torch.from_numpy(plane).cuda()
    u8 = torch.full((33, 80), 0x5A, dtype=torch.uint8, device="cuda")
    api.quantize_device(d, 96, 70, 33, api.SaveMode[mode], u8, 80, api.alloc_scratch(1))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u8[:, :70].cpu().numpy(), oracle.quantize(plane, mode))
    assert (u8[:, 70:].cpu().numpy() == 0x5A).all()


# FilterParams whose responses fit int16 take the packed kernel with runtime
# taps; the others the generic kernel.  Both must equal the oracle.
PARAMS = [(1, 1, 1, 1), (1, 2, 4, 2), (1, 1, 2, 1), (2, 1, 1, 1), (1, 3, 2, 1), (2, 3, 5, 7),
          (3, 1, 1, 2)]


@pytest.mark.parametrize("params", PARAMS)
@pytest.mark.parametrize("pad", [False, True])
def test_params_all_contracts(api, oracle, params, pad):
    import torch
    sys_taps = oracle.make_stream_taps(*params)
    taps = api.Taps.from_dict(sys_taps.as_dict())
    h, w = 203, 301
    img = rand_img(h, w, sum(params), 0xFF)
    ow, oh = (w, h) if pad else (w - 4, h - 4)
    ref = padded_ref(oracle, img, sys_taps) if pad else oracle.run_stream(img, sys_taps)[1]
    d, pitch = to_dev(api, img)
    for planes in (SR, ("u8",), SR + ("u8",)):
        out, op = api.alloc_planes(ow, oh, planes)
        for v in out.values():
            v.fill_(7)
        api.launch_ex(d, pitch, w, h, taps, 1, pad, out, op)
        torch.cuda.synchronize()
        for k in planes:
            want = oracle.clamp_abs(ref["g"]) if k == "u8" else ref[k]
            np.testing.assert_array_equal(out[k][:, :ow].cpu().numpy(), want, err_msg=f"{k} {planes}")
    got = _detect(api, img, pad, api.SaveMode.normalize, planes=("g",), taps=taps)
    np.testing.assert_array_equal(got["g"], ref["g"])
    np.testing.assert_array_equal(got["u8"], oracle.quantize(ref["g"], "normalize"))


def test_fault_injected_runtime_packed(api, oracle):
    """Odd perturbations of the default taps still fit the packed kernel and
    must report recover_diag's ParityViolation with the first pair."""
    import torch
    t = oracle.make_stream_taps()
    t.k0[0] += 1
    taps = api.Taps.from_dict(t.as_dict())
    img = rand_img(40, 70, 5)
    st, _, bad = oracle.run_stream(img, t)
    assert st == 3
    d, pitch = to_dev(api, img)
    out, op = api.alloc_planes(66, 36, SR)
    diag = torch.zeros(8, dtype=torch.int32, device="cuda")
    api.launch(d, pitch, 70, 40, taps, 1, out, op, diag)
    torch.cuda.synchronize()
    assert diag[0].item() > 0


@pytest.mark.parametrize("band", ["8", "32"])
@pytest.mark.parametrize("h,w", [(77, 1541), (9, 129), (40, 515), (3, 600)])
def test_pad_tma_band_loads(api, oracle, monkeypatch, h, w, band):
    """Replicate padding with the TMA band loads (kGeomPadTma, forced by
    SOBEL5_BAND): clamped rows, the left 16-byte lead, right-edge patching."""
    import torch
    monkeypatch.setenv("SOBEL5_BAND", band)
    img = rand_img(h, w, 3 * w + h)
    d, pitch = to_dev(api, img)
    out, op = api.alloc_planes(w, h, SR)
    api.launch_ex(d, pitch, w, h, api.make_stream_taps(), 1, True, out, op)
    torch.cuda.synchronize()
    ref = padded_ref(oracle, img)
    for k in SR:
        np.testing.assert_array_equal(out[k][:, :w].cpu().numpy(), ref[k], err_msg=f"{k} band {band}")
