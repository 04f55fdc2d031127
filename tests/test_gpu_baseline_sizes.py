"""Parity at the BASELINE sizes nothing smaller reaches.

C5: one 32768 x 32768 image on one GPU -- the call ``bench.py --workload
32k-bands`` makes at N=1 -- and the same image as 8 stacked row bands of
4096 rows (the N=8 partition of SURVEY.md section 8e, halos read from the
neighbouring bands' rows), for every output contract:

* SR (4 x int32 + f64) above 300 M output pixels takes 8-row TMA bands, SR32
  takes 12-row bands, the u8 map the packed-float epilogue
  (sobel5_abi.cu, the band rule for big launches);
* rows are compared with the C oracle on sampled windows -- the first and
  last rows (the ragged last band and the last partial wave of CTAs), rows
  across several 8/12-row CTA band boundaries, and the rows around the N=8
  band seams -- on input rows the oracle generates itself (synth_random of
  the window, independent of the device generator);
* the whole 1.07 G-pixel planes are compared ON THE DEVICE between the
  contracts (SR32's integer planes == SR's, |g32 - g| <= 1 ulp of float,
  u8 == clamp_abs(g)) and between the single launch and the 8-band
  partition (bit-identical).

C4: 256 frames of 1920 x 1080 (seed 1 + i) in one sobel5_launch_batch: the
u8 map of EVERY frame hashed against the oracle's, every plane of sampled
frames compared in full.

Oracle: oracle/sobel5_oracle.c via pyoracle (test infrastructure only).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PLANES = ("gx", "gy", "gd", "gdt", "g")
GOLDEN = 0x9E3779B97F4A7C15  # splitmix64 increment (synth.hpp:11-17)


def synth_rows(oracle, w, y0, n, seed):
    """Rows [y0, y0+n) of synth_random(w, H, seed) (synth.hpp:20-35): with
    w % 8 == 0 row y0 starts splitmix64 word y0*w/8, i.e. the same generator
    with the seed advanced by y0*w/8 increments."""
    assert w % 8 == 0
    return oracle.synth_random(w, n, (seed + (y0 * w // 8) * GOLDEN) % (1 << 64))


def oracle_window(oracle, w, oy0, n, seed):
    """Oracle planes of output rows [oy0, oy0+n) (input rows oy0..oy0+n+3)."""
    st, ref, _ = oracle.run_stream(synth_rows(oracle, w, oy0, n + 4, seed))
    assert st == 0
    return ref


def chunks(total, step):
    for y in range(0, total, step):
        yield y, min(total, y + step)


@pytest.fixture(scope="module")
def c5(cuda):
    """The 32K image on the device plus its SR planes (one launch)."""
    import torch
    from paper_2305_00515_b200 import api
    w = h = 32768
    d_in, pitch = api.alloc_input(w, h)
    api.synth_random_device(d_in, pitch, w, h, seed=1)
    out, op = api.alloc_planes(w - 4, h - 4, PLANES)
    diag = torch.zeros(8, dtype=torch.int32, device="cuda")
    api.launch(d_in, pitch, w, h, api.make_stream_taps(), 1, out, op, diag)
    info = api.last_launch()
    # > 300 M output px: 8-row bands of TMA-loaded rows (sobel5_abi.cu)
    assert (info["band"], info["tma_load"], info["kernel"]) == (8, 1, 0), info
    torch.cuda.synchronize()
    assert diag[0].item() == 0
    yield dict(w=w, h=h, d_in=d_in, pitch=pitch, out=out, op=op)
    del out, d_in
    torch.cuda.empty_cache()


def c5_windows(h):
    oh = h - 4
    seam = h // 8  # N = 8 band seams at multiples of 4096 input rows
    return [(0, 30), (seam - 2 - 14, 30), (4 * seam - 2 - 11, 26), (8184, 40),
            (oh - 30, 30)]


def test_c5_input_rows_match_oracle_generator(c5, oracle):
    w = c5["w"]
    for y0, n in [(0, 4), (4094, 8), (c5["h"] - 5, 5)]:
        got = c5["d_in"][y0:y0 + n, :w].cpu().numpy()
        np.testing.assert_array_equal(got, synth_rows(oracle, w, y0, n, 1), err_msg=f"row {y0}")


def test_c5_sr_sampled_rows_vs_oracle(c5, oracle):
    w = c5["w"]
    for oy0, n in c5_windows(c5["h"]):
        ref = oracle_window(oracle, w, oy0, n, 1)
        for k in PLANES:
            got = c5["out"][k][oy0:oy0 + n, : w - 4].cpu().numpy()
            np.testing.assert_array_equal(got, ref[k], err_msg=f"{k} rows {oy0}+{n}")


def test_c5_u8_contract_vs_oracle_and_full_plane(c5, oracle):
    """u8-only launch (the u8 kernel, sobel5_u8.cuh: TMA band rows, packed
    pairs, float epilogue): sampled rows vs the oracle,
    the whole plane vs clamp_abs of the SR launch's g on the device (g has no
    ties at k + 0.5: it is the sqrt of an integer, so round-half-even equals
    std::round)."""
    import torch
    from paper_2305_00515_b200 import api
    w, h = c5["w"], c5["h"]
    out, op = api.alloc_planes(w - 4, h - 4, ("u8",))
    api.launch(c5["d_in"], c5["pitch"], w, h, api.make_stream_taps(), 1, out, op)
    li = api.last_launch()
    # sobel5_u8_kernel, 24-row bands above 96 M output pixels, 4-warp CTAs
    # (1024 columns: 32 column tiles)
    assert li["tma_load"] == 1 and li["band"] == 24 and li["grid_x"] == 32
    torch.cuda.synchronize()
    u8 = out["u8"]
    for oy0, n in c5_windows(h):
        ref = oracle_window(oracle, w, oy0, n, 1)
        np.testing.assert_array_equal(u8[oy0:oy0 + n, : w - 4].cpu().numpy(),
                                      oracle.clamp_abs(ref["g"]), err_msg=f"u8 rows {oy0}+{n}")
    g = c5["out"]["g"]
    for y0, y1 in chunks(h - 4, 2048):
        want = torch.clamp(torch.round(g[y0:y1, : w - 4]), max=255).to(torch.uint8)
        assert torch.equal(u8[y0:y1, : w - 4], want), f"u8 rows {y0}..{y1}"


def test_c5_sr32_contract_full_plane(c5):
    """SR32 (12-row TMA bands above 300 M px): integer planes identical to
    the SR launch's, g32 within 1 ulp of float32 of the double g."""
    import torch
    from paper_2305_00515_b200 import api
    w, h = c5["w"], c5["h"]
    names = ("gx", "gy", "gd", "gdt", "g32")
    out, op = api.alloc_planes(w - 4, h - 4, names)
    api.launch(c5["d_in"], c5["pitch"], w, h, api.make_stream_taps(), 1, out, op)
    info = api.last_launch()
    assert (info["band"], info["tma_load"]) == (12, 1), info
    torch.cuda.synchronize()
    sr = c5["out"]
    for y0, y1 in chunks(h - 4, 4096):
        for k in ("gx", "gy", "gd", "gdt"):
            assert torch.equal(out[k][y0:y1, : w - 4], sr[k][y0:y1, : w - 4]), f"{k} {y0}"
        exact = sr["g"][y0:y1, : w - 4].to(torch.float32)
        ulps = (out["g32"][y0:y1, : w - 4].view(torch.int32).long() -
                exact.view(torch.int32).long()).abs().max().item()
        assert ulps <= 1, f"g32 rows {y0}..{y1}: {ulps} ulp"
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n_bands", [8])
def test_c5_row_bands_equal_single_image(c5, n_bands):
    """The N = 8 row-band partition on one device: each band of 4096 rows
    with its 2-row halos read from the neighbouring bands' rows (the stacked
    kGeomSegTma kernel: CTAs touching a halo row load from global memory,
    the others bulk-copy their rows) stitches to the single launch
    bit-for-bit over the whole image."""
    import torch
    from paper_2305_00515_b200 import api
    from paper_2305_00515_b200.bands import _offset_planes, plan_bands
    w, h, pitch = c5["w"], c5["h"], c5["pitch"]
    d_in = c5["d_in"]
    out, op = api.alloc_planes(w - 4, h - 4, PLANES)
    for r in range(n_bands):
        p = plan_bands(w, h, n_bands, r)
        body = d_in[p.r0:p.r1]
        top = d_in[p.r0 - 2:p.r0] if p.has_top else None
        bot = d_in[p.r1:p.r1 + 2] if p.has_bot else None
        api.launch_band(top, body, bot, pitch, w, p.body_rows, api.make_stream_taps(), 1,
                        _offset_planes(out, p.out_row0, op), op)
        assert api.last_launch()["tma_load"] == 1  # kGeomSegTma
    torch.cuda.synchronize()
    sr = c5["out"]
    for y0, y1 in chunks(h - 4, 4096):
        for k in PLANES:
            assert torch.equal(out[k][y0:y1, : w - 4], sr[k][y0:y1, : w - 4]), f"{k} {y0}"
    del out
    torch.cuda.empty_cache()


def test_c4_batch_256_frames(cuda, oracle):
    """C4: 256 x 1080p (seed 1 + i) in ONE batched launch per contract; the
    u8 map of every frame hashed against the oracle (input hashes too), all
    planes of sampled frames compared in full."""
    import torch
    from paper_2305_00515_b200 import api
    w, h, n = 1920, 1080, 256
    ow, oh = w - 4, h - 4
    d_in, pitch = api.alloc_input(w, h, frames=n)
    for f in range(n):
        api.synth_random_device(d_in[f], pitch, w, h, seed=1 + f)
    taps = api.make_stream_taps()
    sr, op = api.alloc_planes(ow, oh, PLANES, frames=n)
    api.launch_batch(d_in, pitch, h * pitch, w, h, n, taps, 1, sr, op, oh * op)
    info = api.last_launch()
    assert (info["band"], info["tma_load"], info["grid_z"]) == (8, 1, n), info
    u8, op8 = api.alloc_planes(ow, oh, ("u8",), frames=n)
    api.launch_batch(d_in, pitch, h * pitch, w, h, n, taps, 1, u8, op8, oh * op8)
    torch.cuda.synchronize()

    def ref_frame(f):
        img = oracle.synth_random(w, h, 1 + f)
        st, ref, _ = oracle.run_stream(img)
        assert st == 0
        return img, ref

    def check_frame(f):
        img, ref = ref_frame(f)
        assert oracle.fnv1a64(img) == oracle.fnv1a64(
            np.ascontiguousarray(d_in[f, :, :w].cpu().numpy())), f"input frame {f}"
        got = np.ascontiguousarray(u8["u8"][f, :, :ow].cpu().numpy())
        want = oracle.clamp_abs(ref["g"])
        assert oracle.fnv1a64(got) == oracle.fnv1a64(want), f"u8 frame {f}"
        return ref if f in (0, 1, 127, 200, 255) else None

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
        refs = dict(zip(range(n), ex.map(check_frame, range(n))))
    for f, ref in refs.items():
        if ref is None:
            continue
        for k in PLANES:
            np.testing.assert_array_equal(sr[k][f, :, :ow].cpu().numpy(), ref[k],
                                          err_msg=f"frame {f} {k}")
    del sr, u8, d_in
    torch.cuda.empty_cache()
