"""GPU checks of the drop-in's oracle-side API (oracle.hpp) and of its
threading contract.

* conv2d_valid (oracle.hpp:19-49) runs on the device (sobel5_conv2d_valid):
  bit-exact against the C oracle for arbitrary 5x5 / 3x3 int32 kernels,
  including taps at the int32 extremes (the reference's int64 sum cast to
  int32 wraps; the device accumulates mod 2^32);
* sobel5_4d (oracle.hpp:82-98) runs the oracle's own dense algorithm on the
  device (sobel5_dense_4d), bit-exact against the C oracle for default,
  non-default and wide parameter sets -- and therefore an independent check
  of run_stream's streaming kernels;
* run_stream from several host threads at once: each thread gets its own
  context (api.default_context is thread-local, like gpu::thread_context in
  the C++ mirror), results stay bit-exact.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PLANES = ("gx", "gy", "gd", "gdt", "g")


@pytest.fixture(scope="module")
def api(cuda):
    from paper_2305_00515_b200 import api
    return api


@pytest.mark.parametrize("ks", [5, 3])
def test_conv2d_valid_device_vs_oracle(api, oracle, ks):
    rng = np.random.default_rng(ks)
    shapes = [(ks, ks), (ks + 1, 300), (61, 97), (129, 130), (40, 1031), (300, 7)]
    for t, (h, w) in enumerate(shapes * 2):
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        if t % 3 == 0:
            k = rng.integers(-2**31, 2**31, (ks, ks), dtype=np.int64).astype(np.int32)
        else:
            k = rng.integers(-40, 40, (ks, ks)).astype(np.int32)
        np.testing.assert_array_equal(api.conv2d_valid(img, k), oracle.conv2d_valid(img, k),
                                      err_msg=f"{w}x{h} kernel {t}")
    with pytest.raises(api.ImageTooSmall):
        api.conv2d_valid(np.zeros((ks - 1, 20), np.uint8), np.zeros((ks, ks), np.int32))


def test_conv2d_valid_sobel_kernels_equal_run_stream(api, oracle):
    """The materialised Kx..Kdt through conv2d_valid equal run_stream's planes."""
    rng = np.random.default_rng(8)
    img = rng.integers(0, 256, (77, 517), dtype=np.uint8)
    r = api.run_stream(img, api.FilterParams(), api.plan_strips(517, 32, 2), api.Prefetch.on)
    for d, name in enumerate(("gx", "gy", "gd", "gdt")):
        np.testing.assert_array_equal(api.conv2d_valid(img, api.materialize(api.FilterParams(), d)),
                                      getattr(r, name), err_msg=name)


@pytest.mark.parametrize("params", [(1, 2, 6, 4), (2, 3, 5, 1), (1, 32768, 1, 1), (3, 1, 7, 2)])
def test_sobel5_4d_dense_device_vs_oracle(api, oracle, params):
    rng = np.random.default_rng(sum(params))
    for h, w in ((5, 5), (33, 130), (70, 611)):
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        got = api.sobel5_4d(img, api.FilterParams(*params))
        ref = oracle.sobel5_4d(img, *params)
        for k in PLANES:
            np.testing.assert_array_equal(getattr(got, k), ref[k], err_msg=f"{k} {w}x{h}")


def test_run_stream_from_many_threads(api, oracle):
    rng = np.random.default_rng(12)
    imgs = [rng.integers(0, 256, (int(rng.integers(40, 300)), int(rng.integers(40, 700))),
                        dtype=np.uint8) for _ in range(8)]
    results, errors, ctx_ids = {}, [], set()
    lock = threading.Lock()

    def work(i):
        try:
            for rep in range(4):
                img = imgs[(i + rep) % len(imgs)]
                r = api.run_stream(img, api.FilterParams(), api.plan_strips(img.shape[1], 32, 2),
                                   api.Prefetch.on)
                with lock:
                    results[(i, rep)] = (img, r)
                    ctx_ids.add(id(api.default_context()))
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    assert len(ctx_ids) == 6  # one context per thread
    for (img, r) in results.values():
        st, ref, _ = oracle.run_stream(img)
        for k in PLANES:
            np.testing.assert_array_equal(getattr(r, k), ref[k])
