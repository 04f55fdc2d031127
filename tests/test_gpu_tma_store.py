"""GPU parity of the opt-in TMA tensor-store path of the StreamResult
(SOBEL5_TS=1: one CTA stages two rows of its 512-column tile and one thread
writes six cp.async.bulk.tensor boxes; SOBEL5_TS=2: every warp writes its own
128-column boxes; sobel5_packed.cuh kGeomPlainTmaTs / kGeomPlainTmaTw, maps
built by sobel5_tmap.cu).  Bit-exact against the oracle for every plane on
ragged widths (the int32 planes travel as uint64 pairs, so odd widths write
one int32 into the row pitch), odd band tails (the TMA unit clips rows past
out_h) and batches (3-D maps, frame stride)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PLANES = ("gx", "gy", "gd", "gdt", "g")


@pytest.fixture
def ts_env():
    saved = {k: os.environ.get(k) for k in ("SOBEL5_TS", "SOBEL5_BAND")}
    yield
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("band", [2, 8])
@pytest.mark.parametrize("h,w", [(9, 9), (61, 97), (33, 1030), (200, 701), (17, 513), (40, 1029)])
def test_tensor_store_matches_oracle(cuda, oracle, ts_env, mode, band, h, w):
    import torch
    from paper_2305_00515_b200 import api
    os.environ["SOBEL5_TS"] = str(mode)
    os.environ["SOBEL5_BAND"] = str(band)
    img = np.random.default_rng(h * 1000 + w).integers(0, 256, (h, w), dtype=np.uint8)
    d_in, pitch = api.alloc_input(w, h)
    d_in.zero_()
    d_in[:, :w].copy_(torch.from_numpy(img))
    out, op = api.alloc_planes(w - 4, h - 4, PLANES)
    for v in out.values():
        v.fill_(7)
    api.launch(d_in, pitch, w, h, api.make_stream_taps(), 1, out, op)
    torch.cuda.synchronize()
    assert api.last_launch()["tma_load"] == 1 and api.last_launch()["band"] == band
    st, ref, _ = oracle.run_stream(img)
    assert st == 0
    for k in PLANES:
        np.testing.assert_array_equal(out[k][:, : w - 4].cpu().numpy(), ref[k], err_msg=k)


@pytest.mark.parametrize("mode", [1, 2])
def test_tensor_store_batch(cuda, oracle, ts_env, mode):
    import torch
    from paper_2305_00515_b200 import api
    os.environ["SOBEL5_TS"] = str(mode)
    os.environ["SOBEL5_BAND"] = "8"
    w, h, n = 389, 29, 3
    imgs = np.random.default_rng(5).integers(0, 256, (n, h, w), dtype=np.uint8)
    d_in, pitch = api.alloc_input(w, h, frames=n)
    d_in[:, :, :w].copy_(torch.from_numpy(imgs))
    out, op = api.alloc_planes(w - 4, h - 4, PLANES, frames=n)
    api.launch_batch(d_in, pitch, h * pitch, w, h, n, api.make_stream_taps(), 1, out, op,
                     (h - 4) * op)
    torch.cuda.synchronize()
    for f in range(n):
        st, ref, _ = oracle.run_stream(imgs[f])
        for k in PLANES:
            np.testing.assert_array_equal(out[k][f, :, : w - 4].cpu().numpy(), ref[k],
                                          err_msg=f"frame {f} {k}")
