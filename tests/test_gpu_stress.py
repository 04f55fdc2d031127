"""GPU: randomized cross-product of the launch space against the oracle --
image sizes around the lane/warp/CTA tiles, valid and replicate-padded
geometry, every output contract (SR, SR32, u8 alone, mixed subsets), all
four kernel families (default, int16 runtime taps, packed FP32, generic),
prefetch on/off and forced bands (which also force the TMA band loads where
they apply).  Bit-exact, float magnitude within 1 ulp."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PLANE_SETS = [("gx", "gy", "gd", "gdt", "g"), ("gx", "gy", "gd", "gdt", "g32"), ("u8",),
              ("gd", "g"), ("gx", "u8"), ("gy", "gdt", "g", "u8")]
PARAMS = [(1, 2, 6, 4), (1, 1, 1, 1), (2, 3, 5, 7), (1, 32768, 1, 1)]
BANDS = ["", "4", "8", "16", "32"]


@pytest.mark.parametrize("seed", range(int(os.environ.get("SOBEL5_STRESS_SEEDS", "6"))))
def test_random_launch_space(cuda, oracle, monkeypatch, seed):
    import torch
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(1000 + seed)
    for case in range(10):
        w = int(rng.choice([5, 9, 127, 128, 131, 509, 512, 517, 1029, 1543]))
        h = int(rng.integers(5, 90))
        pad = bool(rng.integers(0, 2))
        planes = PLANE_SETS[int(rng.integers(0, len(PLANE_SETS)))]
        prm = PARAMS[int(rng.integers(0, len(PARAMS)))]
        pf = int(rng.integers(0, 2))
        band = BANDS[int(rng.integers(0, len(BANDS)))]
        mask = int(rng.choice([0xFF, 0x0F, 0x03]))
        if band:
            monkeypatch.setenv("SOBEL5_BAND", band)
        else:
            monkeypatch.delenv("SOBEL5_BAND", raising=False)
        # the u8-only kernels' CTA width (sobel5_u8.cuh): default rule or forced
        warps = str(rng.choice(["", "1", "2", "4"]))
        if warps:
            monkeypatch.setenv("SOBEL5_U8_WARPS", warps)
        else:
            monkeypatch.delenv("SOBEL5_U8_WARPS", raising=False)
        img = (rng.integers(0, 256, (h, w), dtype=np.uint8) & mask).astype(np.uint8)
        st_t = oracle.make_stream_taps(*prm)
        taps = api.Taps.from_dict(st_t.as_dict())
        src = img
        if pad:
            st, src = oracle.pad_replicate(img, 2)
            assert st == 0
        st, ref, _ = oracle.run_stream(src, st_t)
        assert st == 0
        ow, oh = (w, h) if pad else (w - 4, h - 4)
        d, pitch = api.alloc_input(w, h)
        d.fill_(0xA5)
        d[:, :w].copy_(torch.from_numpy(img))
        out, op = api.alloc_planes(ow, oh, planes)
        for v in out.values():
            v.fill_(0x5A if v.dtype == torch.uint8 else 7)
        api.launch_ex(d, pitch, w, h, taps, pf, pad, out, op)
        torch.cuda.synchronize()
        what = f"{w}x{h} pad={pad} {planes} {prm} pf={pf} band={band or 'auto'}"
        for k in planes:
            got = out[k][:, :ow].cpu().numpy()
            if k == "u8":
                np.testing.assert_array_equal(got, oracle.clamp_abs(ref["g"]), err_msg=what)
            elif k == "g32":
                exact = ref["g"].astype(np.float32)
                ulps = np.abs(got.view(np.int32).astype(np.int64) - exact.view(np.int32))
                assert ulps.max() <= 1, what
            else:
                np.testing.assert_array_equal(got, ref[k], err_msg=f"{k} {what}")


@pytest.mark.parametrize("seed", range(int(os.environ.get("SOBEL5_STRESS_SEEDS", "6"))))
def test_random_stacked_bands(cuda, oracle, monkeypatch, seed):
    """Stacked row bands ([2 halo rows; body; 2 halo rows], the C5 partition)
    over random sizes, cut points, contracts, kernel families, prefetch and
    forced CTA bands (which switch on kGeomSegTma: body-only CTAs read their
    rows by TMA, halo-touching CTAs from global memory)."""
    import torch
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(5000 + seed)
    for case in range(6):
        w = int(rng.choice([9, 131, 517, 1029, 1543]))
        h = int(rng.integers(12, 120))
        planes = PLANE_SETS[int(rng.integers(0, len(PLANE_SETS)))]
        prm = PARAMS[int(rng.integers(0, 3))]
        pf = int(rng.integers(0, 2))
        band = BANDS[int(rng.integers(0, len(BANDS)))]
        if band:
            monkeypatch.setenv("SOBEL5_BAND", band)
        else:
            monkeypatch.delenv("SOBEL5_BAND", raising=False)
        img = (rng.integers(0, 256, (h, w), dtype=np.uint8) & 0x0F).astype(np.uint8)
        st_t = oracle.make_stream_taps(*prm)
        taps = api.Taps.from_dict(st_t.as_dict())
        st, ref, _ = oracle.run_stream(img, st_t)
        assert st == 0
        r0 = int(rng.integers(0, h // 2))
        r1 = int(rng.integers(max(r0 + 1, h // 2), h + 1))
        body, pitch = api.alloc_input(w, r1 - r0)
        body[:, :w].copy_(torch.from_numpy(img[r0:r1]))
        top = bot = None
        if r0 >= 2:
            top, _ = api.alloc_input(w, 2)
            top[:, :w].copy_(torch.from_numpy(img[r0 - 2:r0]))
        if r1 + 2 <= h:
            bot, _ = api.alloc_input(w, 2)
            bot[:, :w].copy_(torch.from_numpy(img[r1:r1 + 2]))
        stacked = (r1 - r0) + (2 if top is not None else 0) + (2 if bot is not None else 0)
        if stacked < 5:
            continue
        rows = stacked - 4
        out, op = api.alloc_planes(w - 4, rows, planes)
        api.launch_band(top, body, bot, pitch, w, r1 - r0, taps, pf, out, op)
        torch.cuda.synchronize()
        y0 = r0 - 2 if top is not None else r0
        what = f"{w}x{h} rows {r0}:{r1} {planes} {prm} pf={pf} band={band or 'auto'}"
        for k in planes:
            got = out[k][:, :w - 4].cpu().numpy()
            want = ref["g"][y0:y0 + rows] if k in ("u8", "g32") else ref[k][y0:y0 + rows]
            if k == "u8":
                np.testing.assert_array_equal(got, oracle.clamp_abs(want), err_msg=what)
            elif k == "g32":
                ulps = np.abs(got.view(np.int32).astype(np.int64) -
                              want.astype(np.float32).view(np.int32))
                assert ulps.max() <= 1, what
            else:
                np.testing.assert_array_equal(got, want, err_msg=f"{k} {what}")


@pytest.mark.parametrize("seed", range(int(os.environ.get("SOBEL5_STRESS_SEEDS", "6"))))
def test_random_3x3_and_detect(cuda, oracle, monkeypatch, seed):
    """The 3x3 operator (every output subset incl. the u8-only kernel
    sobel3_u8.cuh) and the detect export in both SaveModes (normalize pass 1
    on kernel U's S mode for the default taps), random sizes, padding,
    prefetch, forced bands and u8 CTA widths."""
    import torch
    from paper_2305_00515_b200 import api
    rng = np.random.default_rng(9000 + seed)
    for case in range(8):
        w = int(rng.choice([3, 9, 127, 131, 509, 1029, 2055]))
        h = int(rng.integers(3, 80))
        pad = bool(rng.integers(0, 2))
        pf = int(rng.integers(0, 2))
        band = BANDS[int(rng.integers(0, len(BANDS)))]
        warps = str(rng.choice(["", "1", "2", "4"]))
        for name, val in (("SOBEL5_BAND", band), ("SOBEL5_U8_WARPS", warps)):
            if val:
                monkeypatch.setenv(name, val)
            else:
                monkeypatch.delenv(name, raising=False)
        mask = int(rng.choice([0xFF, 0x0F, 0x03]))
        img = (rng.integers(0, 256, (h, w), dtype=np.uint8) & mask).astype(np.uint8)
        d, pitch = api.alloc_input(w, h)
        d.fill_(0xA5)
        d[:, :w].copy_(torch.from_numpy(img))
        what = f"{w}x{h} pad={pad} pf={pf} band={band or 'auto'} warps={warps or 'auto'}"
        if case % 2 == 0:  # 3x3 operator
            if not pad and (w < 3 or h < 3):
                continue
            planes = [("gx", "gy", "g"), ("u8",), ("gy", "u8"), ("g32",)][int(rng.integers(0, 4))]
            ow, oh = (w, h) if pad else (w - 2, h - 2)
            src = img
            if pad:
                st, src = oracle.pad_replicate(img, 1)
                assert st == 0
            st, ref = oracle.sobel3_2d(src)
            assert st == 0
            out, op = api.alloc_planes(ow, oh, planes)
            for v in out.values():
                v.fill_(0x5A if v.dtype == torch.uint8 else 7)
            api.launch3(d, pitch, w, h, pf, pad, out, op)
            torch.cuda.synchronize()
            for k in planes:
                got = out[k][:, :ow].cpu().numpy()
                if k == "u8":
                    np.testing.assert_array_equal(got, oracle.quantize(ref["g"], "clamp_abs"),
                                                  err_msg=f"3x3 u8 {what}")
                elif k == "g32":
                    exact = ref["g"].astype(np.float32)
                    ulps = np.abs(got.view(np.int32).astype(np.int64) - exact.view(np.int32))
                    assert ulps.max() <= 1, what
                else:
                    np.testing.assert_array_equal(got, ref[k], err_msg=f"3x3 {k} {what}")
        else:  # detect: pad_replicate(img, 2) (optional) -> run_stream -> quantize(g)
            if not pad and (w < 5 or h < 5):
                continue
            mode = api.SaveMode.normalize if rng.integers(0, 2) else api.SaveMode.clamp_abs
            ow, oh = (w, h) if pad else (w - 4, h - 4)
            src = img
            if pad:
                st, src = oracle.pad_replicate(img, 2)
                assert st == 0
            st, ref, _ = oracle.run_stream(src)
            assert st == 0
            out, op = api.alloc_planes(ow, oh, ("u8",))
            out["u8"].fill_(0x5A)
            scratch = api.alloc_scratch(1, "cuda", out_h=oh, pitch=op)
            api.detect_device(d, pitch, w, h, api.make_stream_taps(), pf, pad, mode, out, op,
                              scratch)
            torch.cuda.synchronize()
            want = oracle.quantize(ref["g"], "normalize" if mode == api.SaveMode.normalize
                                   else "clamp_abs")
            np.testing.assert_array_equal(out["u8"][:, :ow].cpu().numpy(), want,
                                          err_msg=f"detect {mode} {what}")
