"""GPU parity of the 3x3 two-direction operator:
run_stream_3x3 (pipeline.hpp:551-573) through the C ABI against the oracle's
sobel3_2d (oracle.hpp:58-70) and the reference fixtures in
tests/golden/sobel3.npz.  gx, gy, g and both u8 exports are bit-exact."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
P3 = ("gx", "gy", "g")
SIZES = [(3, 3), (1, 1), (1, 9), (3, 131), (61, 97), (17, 127), (9, 128), (9, 129), (6, 130),
         (13, 131), (4, 132), (33, 255), (21, 509), (7, 512), (11, 514), (5, 645), (300, 260)]


@pytest.fixture(scope="module")
def api(cuda):
    from paper_2305_00515_b200 import api
    return api


def to_dev(api, img):
    import torch
    h, w = img.shape
    d, pitch = api.alloc_input(w, h)
    d.fill_(0xA5)
    d[:, :w].copy_(torch.from_numpy(np.ascontiguousarray(img)))
    return d, pitch


def ref3(oracle, img, pad):
    if pad:
        st, img = oracle.pad_replicate(img, 1)
        assert st == 0
    st, o = oracle.sobel3_2d(img)
    assert st == 0
    return o


@pytest.mark.parametrize("pad", [False, True])
@pytest.mark.parametrize("prefetch", [0, 1])
@pytest.mark.parametrize("h,w", SIZES)
def test_sobel3_launch(api, oracle, h, w, prefetch, pad):
    import torch
    if not pad and (h < 3 or w < 3):
        pytest.skip("valid mode needs 3x3")
    img = np.random.default_rng(h * 7 + w).integers(0, 256, (h, w), dtype=np.uint8)
    if (h + w) % 3 == 0:
        img &= 0x07
    ow, oh = (w, h) if pad else (w - 2, h - 2)
    d, pitch = to_dev(api, img)
    out, op = api.alloc_planes(ow, oh, P3 + ("u8",))
    for v in out.values():
        v.fill_(7)
    api.launch3(d, pitch, w, h, prefetch, pad, out, op)
    torch.cuda.synchronize()
    ref = ref3(oracle, img, pad)
    for k in P3:
        np.testing.assert_array_equal(out[k][:, :ow].cpu().numpy(), ref[k], err_msg=k)
    np.testing.assert_array_equal(out["u8"][:, :ow].cpu().numpy(), oracle.quantize(ref["g"],
                                                                                   "clamp_abs"))


def test_sobel3_golden_fixtures(api):
    z = np.load(os.path.join(GOLD, "sobel3.npz"))
    names = sorted({k.split("__")[0] for k in z.files})
    assert names
    for n in names:
        r = api.run_stream_3x3(z[f"{n}__img"])
        for k in P3:
            np.testing.assert_array_equal(getattr(r, k), z[f"{n}__{k}"], err_msg=f"{n} {k}")


@pytest.mark.parametrize("prefetch", [0, 1])
def test_run_stream_3x3_api_and_counters(api, oracle, prefetch):
    rng = np.random.default_rng(3)
    for h, w in [(3, 3), (40, 33), (700, 301)]:  # 700 rows: several host chunks
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        plan = api.plan_strips(w, 32, 1)
        r = api.run_stream_3x3(img, plan, api.Prefetch(prefetch))
        ref = ref3(oracle, img, False)
        for k in P3:
            np.testing.assert_array_equal(getattr(r, k), ref[k], err_msg=k)
        assert r.counters == oracle.stream3_counters(h, [s.out_w for s in plan.strips],
                                                     bool(prefetch))
    with pytest.raises(api.ImageTooSmall, match="at least 3x3, got 9x2"):
        api.run_stream_3x3(np.zeros((2, 9), np.uint8))
    with pytest.raises(api.DimMismatch):
        api.run_stream_3x3(np.zeros((9, 9), np.uint8), api.plan_strips(9, 32, 2))


@pytest.mark.parametrize("mode", ["clamp_abs", "normalize"])
@pytest.mark.parametrize("pad", [True, False])
def test_sobel3_detect(api, oracle, pad, mode):
    import torch
    for h, w, mask in [(50, 211, 0xFF), (33, 129, 0x03), (1, 1, 0xFF), (8, 530, 0x01)]:
        if not pad and (h < 3 or w < 3):
            continue
        img = np.random.default_rng(h + w).integers(0, 256, (h, w), dtype=np.uint8) & mask
        ow, oh = (w, h) if pad else (w - 2, h - 2)
        d, pitch = to_dev(api, img)
        out, op = api.alloc_planes(ow, oh, ("g", "u8"))
        api.detect3_device(d, pitch, w, h, 1, pad, api.SaveMode[mode], out, op,
                           api.alloc_scratch(1, out_h=oh, pitch=op))
        torch.cuda.synchronize()
        ref = ref3(oracle, img, pad)
        np.testing.assert_array_equal(out["g"][:, :ow].cpu().numpy(), ref["g"])
        np.testing.assert_array_equal(out["u8"][:, :ow].cpu().numpy(),
                                      oracle.quantize(ref["g"], mode), err_msg=f"{h}x{w}")
