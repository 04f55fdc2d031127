"""GPU parity of the u8-only instantiations (the clamp_abs edge map written
alone).  These kernels replace the integer extraction + integer sum of
squares of the other contracts with a packed-FP32 epilogue
(sobel5_packed.cuh: pair_to_float2 / sumsq4 / u8_from_sf2), so they are
checked on their own: the 5x5 valid and replicate-padded geometries, the
batch launch, the 3x3 operator, against the oracle's clamp_abs(g)
(image_io.hpp:235-240) and the reference's full-size FNV-1a u8 hashes.
Low-amplitude inputs (masks 0x01..0x0f) keep most pixels below the 255
saturation so the rounding path is exercised; bit-exact throughout."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "hashes.json")) as f:
    HASHES = json.load(f)
SIZES = [(5, 5), (6, 9), (61, 97), (17, 127), (9, 128), (9, 129), (13, 131), (33, 255),
         (21, 509), (7, 512), (11, 513), (5, 645), (300, 260), (150, 700)]
MASKS = [0xFF, 0x0F, 0x07, 0x03, 0x01]


@pytest.fixture(scope="module")
def api(cuda):
    from paper_2305_00515_b200 import api
    return api


def img_of(h, w, seed, mask):
    return (np.random.default_rng(seed).integers(0, 256, (h, w), dtype=np.uint8) & mask).astype(
        np.uint8)


def to_dev(api, img):
    import torch
    h, w = img.shape
    d, pitch = api.alloc_input(w, h)
    d.fill_(0xA5)  # poison past the width
    d[:, :w].copy_(torch.from_numpy(np.ascontiguousarray(img)))
    return d, pitch


@pytest.mark.parametrize("prefetch", [0, 1])
@pytest.mark.parametrize("h,w", SIZES)
def test_u8_only_valid(api, oracle, h, w, prefetch):
    import torch
    for k, mask in enumerate(MASKS):
        img = img_of(h, w, 97 * h + w + k, mask)
        d, pitch = to_dev(api, img)
        out, op = api.alloc_planes(w - 4, h - 4, ("u8",))
        out["u8"].fill_(0x5A)
        api.launch(d, pitch, w, h, api.make_stream_taps(), prefetch, out, op)
        torch.cuda.synchronize()
        st, ref, _ = oracle.run_stream(img)
        assert st == 0
        np.testing.assert_array_equal(out["u8"][:, : w - 4].cpu().numpy(),
                                      oracle.clamp_abs(ref["g"]), err_msg=f"mask {mask:#x}")


@pytest.mark.parametrize("h,w", [(1, 1), (2, 3), (5, 5), (61, 97), (9, 129), (33, 255),
                                 (7, 512), (300, 260)])
def test_u8_only_pad(api, oracle, h, w):
    import torch
    for k, mask in enumerate(MASKS):
        img = img_of(h, w, 31 * h + w + k, mask)
        d, pitch = to_dev(api, img)
        out, op = api.alloc_planes(w, h, ("u8",))
        out["u8"].fill_(0x5A)
        scratch = api.alloc_scratch(1, out_h=h, pitch=op)
        api.detect_device(d, pitch, w, h, api.make_stream_taps(), 1, True,
                          api.SaveMode.clamp_abs, out, op, scratch)
        torch.cuda.synchronize()
        st, padded = oracle.pad_replicate(img, 2)
        st, ref, _ = oracle.run_stream(padded)
        assert st == 0
        np.testing.assert_array_equal(out["u8"][:, :w].cpu().numpy(),
                                      oracle.clamp_abs(ref["g"]), err_msg=f"mask {mask:#x}")


def test_u8_only_batch(api, oracle):
    import torch
    w, h, n = 389, 29, 6
    imgs = np.stack([img_of(h, w, 500 + f, MASKS[f % len(MASKS)]) for f in range(n)])
    d_in, pitch = api.alloc_input(w, h, frames=n)
    d_in[:, :, :w].copy_(torch.from_numpy(imgs))
    out, op = api.alloc_planes(w - 4, h - 4, ("u8",), frames=n)
    api.launch_batch(d_in, pitch, h * pitch, w, h, n, api.make_stream_taps(), 1, out, op,
                     (h - 4) * op)
    torch.cuda.synchronize()
    for f in range(n):
        st, ref, _ = oracle.run_stream(imgs[f])
        np.testing.assert_array_equal(out["u8"][f, :, : w - 4].cpu().numpy(),
                                      oracle.clamp_abs(ref["g"]), err_msg=f"frame {f}")


@pytest.mark.parametrize("key", list(HASHES))
def test_u8_only_golden_hashes_full_size(api, oracle, key):
    """C1..C3 full-size clamp_abs maps vs the reference's FNV-1a hashes."""
    import torch
    e = HASHES[key]
    w, h = e["w"], e["h"]
    d_in, pitch = api.alloc_input(w, h)
    api.synth_random_device(d_in, pitch, w, h, e["seed"], e["mask"])
    out, op = api.alloc_planes(w - 4, h - 4, ("u8",))
    api.launch(d_in, pitch, w, h, api.make_stream_taps(), 1, out, op)
    torch.cuda.synchronize()
    host = np.ascontiguousarray(out["u8"][:, : w - 4].cpu().numpy())
    assert f"{oracle.fnv1a64(host):016x}" == e["fnv1a64"]["u8"]


@pytest.mark.parametrize("pad", [False, True])
@pytest.mark.parametrize("h,w", [(3, 3), (1, 9), (61, 97), (9, 129), (33, 255), (7, 512),
                                 (300, 260)])
def test_sobel3_u8_only(api, oracle, h, w, pad):
    import torch
    if not pad and (h < 3 or w < 3):
        pytest.skip("valid mode needs 3x3")
    for k, mask in enumerate(MASKS):
        img = img_of(h, w, 13 * h + w + k, mask)
        ow, oh = (w, h) if pad else (w - 2, h - 2)
        d, pitch = to_dev(api, img)
        out, op = api.alloc_planes(ow, oh, ("u8",))
        out["u8"].fill_(0x5A)
        api.launch3(d, pitch, w, h, 1, pad, out, op)
        torch.cuda.synchronize()
        src = img
        if pad:
            st, src = oracle.pad_replicate(img, 1)
            assert st == 0
        st, ref = oracle.sobel3_2d(src)
        assert st == 0
        np.testing.assert_array_equal(out["u8"][:, :ow].cpu().numpy(),
                                      oracle.quantize(ref["g"], "clamp_abs"),
                                      err_msg=f"mask {mask:#x}")


@pytest.mark.parametrize("warps", ["1", "2", "4"])
@pytest.mark.parametrize("band", ["4", "13", "32"])
@pytest.mark.parametrize("op", [5, 3])
@pytest.mark.parametrize("pad", [False, True])
def test_u8_kernels_every_cta_width_and_band(api, oracle, monkeypatch, warps, band, op, pad):
    """The u8-only kernels (sobel5_u8.cuh, sobel3_u8.cuh) at every CTA width
    (1, 2, 4 warps: 256 / 512 / 1024 columns) and band height the size rules
    can pick or a caller can force, valid and padded, on a ragged image that
    spans several column tiles and a partial last band."""
    import torch
    monkeypatch.setenv("SOBEL5_U8_WARPS", warps)
    monkeypatch.setenv("SOBEL5_BAND", band)
    h, w = 157, 2333
    for k, mask in enumerate((0xFF, 0x07)):
        img = img_of(h, w, 7 * k + op, mask)
        r = (op - 1) // 2
        ow, oh = (w, h) if pad else (w - 2 * r, h - 2 * r)
        d, pitch = to_dev(api, img)
        out, op_ = api.alloc_planes(ow, oh, ("u8",))
        out["u8"].fill_(0x5A)
        if op == 5:
            api.launch_ex(d, pitch, w, h, api.make_stream_taps(), 1, pad, out, op_)
        else:
            api.launch3(d, pitch, w, h, 1, pad, out, op_)
        torch.cuda.synchronize()
        src = img
        if pad:
            st, src = oracle.pad_replicate(img, r)
            assert st == 0
        if op == 5:
            st, ref, _ = oracle.run_stream(src)
            want = oracle.clamp_abs(ref["g"])
        else:
            st, ref = oracle.sobel3_2d(src)
            want = oracle.quantize(ref["g"], "clamp_abs")
        assert st == 0
        np.testing.assert_array_equal(out["u8"][:, :ow].cpu().numpy(), want,
                                      err_msg=f"op {op} mask {mask:#x}")
