"""CPU: the product library loads, exports its ABI, and its host-side logic
(taps, validation, strips, counters) matches the reference's known answers.
No compute entry point is exercised here beyond checking that it fails
loudly (never silently computes on the CPU) when no GPU is present."""
import ctypes as C
import json
import os
import re
from fractions import Fraction

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
with open(os.path.join(GOLD, "known.json")) as f:
    KNOWN = json.load(f)

# reference error classes as numbered by oracle/ref_shim.cpp
REF_ERR = {10: "NonPositiveParam", 11: "NonIntegralWeight", 12: "ParamOverflow",
           13: "ImageTooSmall", 14: "RowTooShort", 17: "ParityViolation",
           18: "LaneTooNarrow", 19: "DimMismatch"}


@pytest.fixture(scope="module")
def S():
    import paper_2305_00515_b200 as S
    return S


@pytest.fixture(scope="module")
def lib():
    from paper_2305_00515_b200 import _abi
    return _abi.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sobel5_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sobel[35]_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(lib):
    from paper_2305_00515_b200 import _abi
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/sobel5_gpu.h but not exported"
    assert set(syms) == set(_abi.EXPORTS)


def test_library_is_sm100a(lib):
    """The shipped .so carries sm_100a SASS (no PTX-only or other-arch path)."""
    import subprocess
    from paper_2305_00515_b200 import _abi
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.lib_path()], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_abi_version_and_status_strings(lib):
    assert lib.sobel5_abi_version() == 1
    assert lib.sobel5_status_string(0) == b"ok"
    assert b"odd" in lib.sobel5_status_string(3)


def test_make_taps_matches_reference(S):
    assert S.make_stream_taps().as_dict() == KNOWN["default_taps"]
    for params, t in KNOWN["taps"].items():
        a, b, m, n = eval(params)
        if "error" in t:
            with pytest.raises(S.Error):
                S.make_stream_taps(S.FilterParams(a, b, m, n))
        else:
            assert S.make_stream_taps(S.FilterParams(a, b, m, n)).as_dict() == t, params


def test_validate_params_errors_and_messages(S):
    for key, e in KNOWN["errors"].items():
        a, b, m, n = json.loads(key)
        p = S.FilterParams(a, Fraction(*b), Fraction(*m), Fraction(*n))
        if e["code"] == 0:
            assert S.make_stream_taps(p).as_dict() == e["taps"]
            continue
        cls = getattr(S, REF_ERR[e["code"]])
        with pytest.raises(cls) as ei:
            S.validate_params(p)
        assert str(ei.value) == e["message"], key


def test_c_abi_param_errors(lib):
    from paper_2305_00515_b200._abi import NON_POSITIVE_PARAM, PARAM_OVERFLOW, Taps
    t = Taps()
    assert lib.sobel5_make_taps(0, 2, 6, 4, C.byref(t)) == NON_POSITIVE_PARAM
    assert lib.sobel5_make_taps(1, 65536, 1, 1, C.byref(t)) == PARAM_OVERFLOW
    assert lib.sobel5_make_taps(1, 200, 200, 1, C.byref(t)) == PARAM_OVERFLOW
    assert lib.sobel5_make_taps(1, 32768, 1, 1, C.byref(t)) == 0 and t.wide_vagg == 1


def test_materialize_matches_reference(S):
    for params, ks in KNOWN["kernels"].items():
        p = S.FilterParams(*eval(params))
        for d in range(4):
            np.testing.assert_array_equal(S.materialize(p, d), ks[d])


def test_plan_strips_matches_reference(S):
    for key, e in KNOWN["strips"].items():
        parts = [int(x) for x in key.split(",")]
        w, lanes = parts[0], parts[1]
        r = parts[2] if len(parts) > 2 else 2
        if e["code"]:
            with pytest.raises(getattr(S, REF_ERR[e["code"]])) as ei:
                S.plan_strips(w, lanes, r)
            assert str(ei.value) == e["message"]
        else:
            plan = S.plan_strips(w, lanes, r)
            assert [(s.in_off, s.out_off, s.out_w) for s in plan.strips] == \
                [tuple(s) for s in e["strips"]]


def test_strip_coverage_exhaustive(S):
    """SPEC ACCEPTANCE 8 (sampled widths): disjoint exhaustive output ranges,
    2r input overlap between neighbours."""
    for w in list(range(5, 300)) + [1023, 2048, 4096]:
        for lanes in (8, 16, 32, 64):
            plan = S.plan_strips(w, lanes, 2)
            covered = 0
            for i, s in enumerate(plan.strips):
                assert s.out_off == covered and s.in_off == s.out_off
                covered += s.out_w
                if i:
                    prev = plan.strips[i - 1]
                    assert prev.in_off + prev.out_w + 4 - s.in_off == 4
            assert covered == w - 4


def test_plan_counters_match_reference(S):
    taps = S.make_stream_taps()
    for key, c in KNOWN["counters"].items():
        dims, lanes, pf = key.split(",")
        w, h = map(int, dims.split("x"))
        plan = S.plan_strips(w, int(lanes), 2)
        assert S.plan_counters(h, plan, taps, S.Prefetch(int(pf))) == c, key
    # SPEC ACCEPTANCE 4 / SURVEY A.2: (k0 + k1) per strip per row ~ 3, 25% below 4
    c = KNOWN["counters"]["1024x1024,32,1"]
    assert (c["row_conv5_k0"] + c["row_conv5_k1"]) / 37 / 1024 == pytest.approx(3.0, abs=0.01)


def test_run_stream_validation_before_compute(S):
    """run_stream checks size, then plan, before touching the GPU
    (pipeline.hpp:454-460)."""
    with pytest.raises(S.ImageTooSmall) as ei:
        S.run_stream(np.zeros((4, 9), np.uint8), S.FilterParams(), S.plan_strips(9, 32, 2),
                     S.Prefetch.on)
    assert str(ei.value) == "streaming filter needs at least 5x5, got 9x4"
    with pytest.raises(S.DimMismatch) as ei:
        S.run_stream(np.zeros((9, 9), np.uint8), S.FilterParams(), S.plan_strips(10, 32, 2),
                     S.Prefetch.on)
    assert str(ei.value) == "strip plan covers 10 columns at radius 2, image has 9"


def test_no_silent_cpu_fallback_without_gpu(lib):
    """Without a device every compute entry point reports an error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2305_00515_b200._abi import NO_DEVICE, OK
    h = C.c_void_p()
    assert lib.sobel5_ctx_create(C.byref(h), 0) == NO_DEVICE
    from paper_2305_00515_b200._abi import Planes, Taps
    t = Taps()
    lib.sobel5_make_taps(1, 2, 6, 4, C.byref(t))
    buf = (C.c_uint8 * 4096)()
    out = (C.c_int32 * 4096)()
    addr = (C.addressof(buf) + 15) // 16 * 16
    oaddr = (C.addressof(out) + 31) // 32 * 32
    pl = Planes(gx=oaddr, pitch=32)
    st = lib.sobel5_launch(addr, 64, 32, 16, C.byref(t), 1, C.byref(pl), None, None)
    assert st != OK


def test_kernel_selection_by_taps_bound():
    """sobel5_kernel_for_taps (host-only): default taps -> packed default
    algebra; responses < 2^15 -> packed int16 lanes with runtime taps; partial
    sums < 2^22 -> packed FP32; anything else -> generic 32-bit kernel."""
    from paper_2305_00515_b200 import api
    cases = {(1, 2, 6, 4): "packed_default", (1, 1, 1, 1): "packed_runtime_taps",
             (2, 3, 5, 1): "packed_runtime_taps", (2, 3, 5, 7): "f32x2_runtime_taps",
             (2, 5, 11, 13): "f32x2_runtime_taps", (1, 32768, 1, 1): "generic",
             (4, 16, 64, 64): "generic"}
    for prm, want in cases.items():
        assert api.kernel_for(api.make_stream_taps(api.FilterParams(*prm))) == want, prm
    t = api.make_stream_taps()
    t.k0[0] += 2  # fault injection keeps the int16 bound
    assert api.kernel_for(t) == "packed_runtime_taps"
    t.k1[2] = 1 << 24  # a tap not exact in FP32 is never given to the f32 kernel
    assert api.kernel_for(t) == "generic"


def test_python_synth_random_matches_reference_generator(oracle):
    """api.synth_random (host numpy, synth.hpp:20-35) == the C oracle's, and
    the SURVEY A.2 known answer."""
    import numpy as np
    from paper_2305_00515_b200 import api
    assert api.synth_random(16, 1, 1).ravel().tolist() == [
        193, 92, 2, 137, 236, 45, 10, 145, 103, 236, 142, 101, 161, 141, 235, 190]
    for w, h, seed in ((1920, 1080, 1), (333, 17, 9), (5, 5, 123)):
        assert np.array_equal(api.synth_random(w, h, seed), oracle.synth_random(w, h, seed))
