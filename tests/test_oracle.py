"""CPU: pin the C oracle against the reference's golden vectors.

The oracle (oracle/sobel5_oracle.c) is only trusted after it reproduces
(1) the fixtures generated from the reference itself (tests/golden/,
made by tests/golden/make_golden.py from oracle/_ref), (2) the SURVEY.md
Appendix A.3 FNV-1a hashes, and (3) live outputs of the compiled reference
where it is available.
"""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PLANES = ("gx", "gy", "gd", "gdt", "g")


def load_cases():
    with open(os.path.join(GOLD, "cases.json")) as f:
        meta = json.load(f)
    arrs = np.load(os.path.join(GOLD, "cases.npz"))
    return meta, arrs


CASES, ARRS = load_cases()
with open(os.path.join(GOLD, "known.json")) as f:
    KNOWN = json.load(f)
with open(os.path.join(GOLD, "hashes.json")) as f:
    HASHES = json.load(f)


@pytest.mark.parametrize("i", range(len(CASES)), ids=[c["name"] for c in CASES])
def test_oracle_run_stream_matches_reference_fixture(oracle, i):
    import pyoracle
    c = CASES[i]
    taps = pyoracle.Taps.from_dict(c["taps"])
    st, out, bad = oracle.run_stream(ARRS[f"img{i}"], taps)
    if c["status"] == 13:  # ImageTooSmall
        assert st == 1
        return
    if c["status"] == 17:  # ParityViolation, message carries the first pair
        assert st == 3
        assert c["message"] == f"odd sum/difference pair ({bad[0]}, {bad[1]})"
        return
    assert st == 0
    for k in PLANES:
        np.testing.assert_array_equal(out[k], ARRS[f"{k}{i}"], err_msg=k)
    np.testing.assert_array_equal(oracle.clamp_abs(out["g"]), ARRS[f"u8{i}"])


@pytest.mark.parametrize("i", [i for i, c in enumerate(CASES)
                               if c["status"] == 0 and not c["name"].startswith("fault")],
                         ids=lambda i: CASES[i]["name"])
def test_oracle_sobel5_4d_equals_stream_fixture(oracle, i):
    """oracle.hpp sobel5_4d == pipeline.hpp run_stream (SPEC oracle equivalence)."""
    c = CASES[i]
    out = oracle.sobel5_4d(ARRS[f"img{i}"], *c["params"])
    for k in PLANES:
        np.testing.assert_array_equal(out[k], ARRS[f"{k}{i}"], err_msg=k)


@pytest.mark.parametrize("key", [k for k in HASHES if k.startswith("1920x1080")])
def test_oracle_golden_hashes_c1(oracle, key):
    e = HASHES[key]
    img = oracle.synth_random(e["w"], e["h"], e["seed"]) & e["mask"]
    assert f"{oracle.fnv1a64(img):016x}" == e["fnv1a64"]["input"]
    st, out, _ = oracle.run_stream(img)
    assert st == 0
    for k in PLANES:
        assert f"{oracle.fnv1a64(out[k]):016x}" == e["fnv1a64"][k], k
    assert f"{oracle.fnv1a64(oracle.clamp_abs(out['g'])):016x}" == e["fnv1a64"]["u8"]


def test_oracle_synth_random_known_answer(oracle):
    # synth_random(16,1,seed=1)
    assert oracle.synth_random(16, 1, 1).ravel().tolist() == KNOWN["synth16"]


def test_oracle_taps_match_reference(oracle):
    assert oracle.make_stream_taps().as_dict() == KNOWN["default_taps"]
    for params, t in KNOWN["taps"].items():
        if "error" in t:
            continue
        assert oracle.make_stream_taps(*eval(params)).as_dict() == t, params


def test_oracle_kernels_match_reference(oracle):
    for params, ks in KNOWN["kernels"].items():
        for d in range(4):
            np.testing.assert_array_equal(oracle.materialize(*eval(params), d), ks[d])


def test_oracle_counters_match_reference(oracle):
    for key, c in KNOWN["counters"].items():
        dims, lanes, pf = key.split(",")
        w, h = map(int, dims.split("x"))
        strips = KNOWN["strips"].get(f"{w},{lanes}")
        if strips is None:
            step = int(lanes) - 4
            widths = [min(step, (w - 4) - off) for off in range(0, w - 4, step)]
        else:
            widths = [s[2] for s in strips["strips"]]
        assert oracle.stream_counters(h, widths, prefetch=bool(int(pf))) == c, key


def test_spec_examples(oracle):
    """SPEC.md per-op examples."""
    ramp = np.tile(np.arange(5, dtype=np.uint8), (5, 1))
    st, o, _ = oracle.run_stream(ramp)
    assert (o["gx"][0, 0], o["gy"][0, 0], o["gd"][0, 0], o["gdt"][0, 0]) == (128, 0, 96, -96)
    assert o["g"][0, 0] == 186.59046063504962
    st, o, _ = oracle.run_stream(np.full((9, 9), 7, np.uint8))
    assert all(not o[k].any() for k in PLANES)
    imp = np.zeros((9, 9), np.uint8)
    imp[4, 4] = 1
    st, o, _ = oracle.run_stream(imp)
    assert o["gd"][0].tolist() == [6, 4, 1, 2, 0]  # 180-degree flipped Kd row
    step = np.zeros((5, 5), np.uint8)
    step[:, 3:] = 255
    st, o, _ = oracle.run_stream(step)
    assert o["gx"][0, 0] == 12240
    # linearity in a (SPEC sobel5_4d: params (2,2,6,4) doubles every plane)
    rng = np.random.default_rng(1)
    img = rng.integers(0, 256, (20, 20), dtype=np.uint8)
    o1, o2 = oracle.sobel5_4d(img), oracle.sobel5_4d(img, 2, 2, 6, 4)
    for k in PLANES:
        np.testing.assert_array_equal(o2[k], 2 * o1[k])


def test_oracle_vs_compiled_reference_random(oracle, reference):
    """Live cross-check against the reference headers (ACCEPTANCE 1 style)."""
    import pyoracle
    rng = np.random.default_rng(7)
    for trial in range(40):
        w, h = int(rng.integers(5, 160)), int(rng.integers(5, 90))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        if trial % 4 == 0:
            img &= 7
        lanes = int(rng.choice([8, 16, 32, 64]))
        code, ref, _, msg = reference.run_stream(img, lanes=lanes, prefetch=bool(trial % 2))
        assert code == 0, msg
        st, out, _ = oracle.run_stream(img, pyoracle.Taps.from_dict(KNOWN["default_taps"]))
        for k in PLANES:
            np.testing.assert_array_equal(out[k], ref[k], err_msg=f"{k} {w}x{h}")


def test_conv2d_valid_restatement_matches_reference(oracle, reference):
    """oracle_conv2d_valid / _valid3 (oracle.hpp:19-49) against the compiled
    reference for arbitrary 5x5 and 3x3 kernels, int32 extremes included
    (the int64 sum's cast to int32 wraps)."""
    rng = np.random.default_rng(21)
    for ks in (5, 3):
        for t in range(24):
            img = rng.integers(0, 256, (int(rng.integers(ks, 40)), int(rng.integers(ks, 70))),
                               dtype=np.uint8)
            if t % 3 == 0:
                k = rng.integers(-2**31, 2**31, (ks, ks), dtype=np.int64).astype(np.int32)
            else:
                k = rng.integers(-60, 60, (ks, ks)).astype(np.int32)
            st, ref = reference.conv2d_valid(img, k)
            assert st == 0
            np.testing.assert_array_equal(oracle.conv2d_valid(img, k), ref)
        st, _ = reference.conv2d_valid(np.zeros((ks - 1, 9), np.uint8), np.zeros((ks, ks), np.int32))
        assert st == 13  # ImageTooSmall
