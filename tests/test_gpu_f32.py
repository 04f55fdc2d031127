"""GPU parity of the packed-FP32 runtime-taps kernel (sobel5_f32x2.cuh): the
FilterParams whose responses overflow the int16 lanes but stay below 2^22,
and fault-injected taps in that range, through every geometry (valid,
replicate-padded, stacked row bands, batches) and both magnitude modes
(exact 32-bit S and exact 64-bit S), bit-exact against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SR = ("gx", "gy", "gd", "gdt", "g")
F32_PARAMS = [(2, 3, 5, 7), (3, 2, 7, 5), (1, 4, 9, 9), (2, 5, 11, 13), (1, 8, 8, 8)]


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


def img_of(h, w, seed, mask=0xFF):
    return (np.random.default_rng(seed).integers(0, 256, (h, w), dtype=np.uint8) & mask).astype(
        np.uint8)


def test_params_select_the_f32_kernel(api, oracle):
    for prm in F32_PARAMS:
        t = api.Taps.from_dict(oracle.make_stream_taps(*prm).as_dict())
        assert api.kernel_for(t) == "f32x2_runtime_taps", prm


@pytest.mark.parametrize("prefetch", [0, 1])
@pytest.mark.parametrize("params", F32_PARAMS)
@pytest.mark.parametrize("h,w", [(5, 5), (9, 133), (40, 515), (23, 37), (130, 777)])
def test_f32_valid(api, oracle, h, w, params, prefetch):
    import torch
    st_t = oracle.make_stream_taps(*params)
    taps = api.Taps.from_dict(st_t.as_dict())
    for k, mask in enumerate((0xFF, 0x0F)):
        img = img_of(h, w, 5 * h + w + k, mask)
        d, pitch = to_dev(api, img)
        out, op = api.alloc_planes(w - 4, h - 4, SR + ("u8",))
        for v in out.values():
            v.fill_(7)
        diag = torch.zeros(8, dtype=torch.int32, device="cuda")
        api.launch(d, pitch, w, h, taps, prefetch, out, op, diag)
        torch.cuda.synchronize()
        st, ref, _ = oracle.run_stream(img, st_t)
        assert st == 0 and diag[0].item() == 0
        for p in SR:
            np.testing.assert_array_equal(out[p][:, : w - 4].cpu().numpy(), ref[p], err_msg=p)
        np.testing.assert_array_equal(out["u8"][:, : w - 4].cpu().numpy(),
                                      oracle.clamp_abs(ref["g"]))


@pytest.mark.parametrize("params", F32_PARAMS[:3])
@pytest.mark.parametrize("h,w", [(1, 1), (9, 129), (61, 97)])
def test_f32_pad(api, oracle, h, w, params):
    import torch
    st_t = oracle.make_stream_taps(*params)
    taps = api.Taps.from_dict(st_t.as_dict())
    img = img_of(h, w, 11 + h * w)
    d, pitch = to_dev(api, img)
    out, op = api.alloc_planes(w, h, SR)
    api.launch_ex(d, pitch, w, h, taps, 1, True, out, op)
    torch.cuda.synchronize()
    st, padded = oracle.pad_replicate(img, 2)
    st, ref, _ = oracle.run_stream(padded, st_t)
    for p in SR:
        np.testing.assert_array_equal(out[p][:, :w].cpu().numpy(), ref[p], err_msg=p)


def test_f32_bands_and_batch(api, oracle):
    import torch
    st_t = oracle.make_stream_taps(2, 3, 5, 7)
    taps = api.Taps.from_dict(st_t.as_dict())
    h, w = 41, 301
    img = img_of(h, w, 77)
    st, ref, _ = oracle.run_stream(img, st_t)
    # two stacked bands with 2-row halos == the whole image
    d, pitch = to_dev(api, img)
    cut = 20
    for r0, r1 in ((0, cut), (cut, h)):
        top = d[r0 - 2] if r0 > 0 else None
        bot = d[r1] if r1 < h else None
        body = d[r0:r1]
        rows = (r1 - r0) + (2 if top is not None else 0) + (2 if bot is not None else 0)
        out, op = api.alloc_planes(w - 4, rows - 4, SR)
        api.launch_band(top, body, bot, pitch, w, r1 - r0, taps, 1, out, op)
        torch.cuda.synchronize()
        o0 = r0 - 2 if top is not None else 0
        for p in SR:
            np.testing.assert_array_equal(out[p][:, : w - 4].cpu().numpy(),
                                          ref[p][o0:o0 + rows - 4], err_msg=f"band {r0} {p}")
    # batch of frames
    n = 3
    imgs = np.stack([img_of(h, w, 200 + f) for f in range(n)])
    d_in, pitch = api.alloc_input(w, h, frames=n)
    d_in[:, :, :w].copy_(torch.from_numpy(imgs))
    out, op = api.alloc_planes(w - 4, h - 4, SR, frames=n)
    api.launch_batch(d_in, pitch, h * pitch, w, h, n, taps, 1, out, op, (h - 4) * op)
    torch.cuda.synchronize()
    for f in range(n):
        st, ref, _ = oracle.run_stream(imgs[f], st_t)
        for p in SR:
            np.testing.assert_array_equal(out[p][f, :, : w - 4].cpu().numpy(), ref[p],
                                          err_msg=f"frame {f} {p}")


def test_f32_fault_injected_parity_violation(api, oracle):
    """Fault-injected (2,3,5,7) taps still in FP32 range: the odd P+M is
    reported like the reference's ParityViolation; an even fault computes
    the reference's planes."""
    import torch
    img = img_of(30, 90, 5)
    for delta, odd in ((1, True), (2, False)):
        st_t = oracle.make_stream_taps(2, 3, 5, 7)
        st_t.k1[2] += delta
        taps = api.Taps.from_dict(st_t.as_dict())
        assert api.kernel_for(taps) == "f32x2_runtime_taps"
        d, pitch = to_dev(api, img)
        out, op = api.alloc_planes(86, 26, SR)
        diag = torch.zeros(8, dtype=torch.int32, device="cuda")
        api.launch(d, pitch, 90, 30, taps, 1, out, op, diag)
        torch.cuda.synchronize()
        st, ref, bad = oracle.run_stream(img, st_t)
        if odd:
            assert st == 3 and diag[0].item() > 0  # oracle status 3: parity violation
            P, M = diag[6].item(), diag[7].item()  # sobel5_diag.sum, .diff
            assert (P + M) % 2 != 0
            assert (P, M) == bad  # the first odd pixel in row-major order (one strip)
        else:
            assert st == 0 and diag[0].item() == 0
            for p in SR:
                np.testing.assert_array_equal(out[p][:, :86].cpu().numpy(), ref[p], err_msg=p)
