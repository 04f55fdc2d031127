"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Everything here is produced by oracle/_ref/libsobel5_ref.so, i.e. the
reference's own headers (pipeline.hpp run_stream, oracle.hpp sobel5_4d,
filter_algebra.hpp, strips.hpp, synth.hpp) compiled unmodified.  The only
restated piece is clamp_abs (image_io.hpp:235-240, not compilable here
because that header needs libpng); it is applied to the reference's g plane
by the C oracle and cross-checked against SURVEY.md Appendix A.3.

Outputs:
  cases.npz      small input/output cases (inputs, taps, reference planes)
  cases.json     metadata for cases.npz
  hashes.json    FNV-1a-64 of the full-size planes at configs C1..C3
  known.json     host-side known answers (taps, kernels, strips, errors,
                 counters, row helpers)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle  # noqa: E402

PLANES = ("gx", "gy", "gd", "gdt", "g")

# SURVEY.md Appendix A.3 (oracle sobel5_4d, default params, synth_random seed 1)
SURVEY_A3 = {
    "1920x1080/ff": "c0f4f3dd50a5dde6 46506dea3f58aa67 103f40bace0f4c67 748f2dff2766815e "
                    "9d5091c02c2c44cb 4066babdad7b6b8d 6d5379a2e61bc08f",
    "1920x1080/0f": "ae9ea6c49161d786 573658b868d2aeec 4a6d9d5fdbc9a63c 8c4f321ec9151c62 "
                    "c5b6fbef33225049 6cb45987ac98b8cd eefaa4d994801e0c",
    "1920x1080/07": "906c6c501a48c45e adcd7eec63ac760c b44f18786465cfc9 0285aabae226ecf7 "
                    "83d15d5c941e96c6 2792958ace2bca14 1d0cdd8dfd36419b",
    "3840x2160/ff": "ad0678d022cf56c4 1a1f5fb2b7b883b8 5c426c01134459bc 100216b42ce567eb "
                    "b8c3cfab3fd77277 7f8a6095a3f9e7fb f231f00e0fa19076",
    "3840x2160/07": "6058f564c650d1d4 afb0e6efb1d7c495 750daab657ba16d1 39241b6a8ca18169 "
                    "a1b8be8d12a17a65 ebfadfe35bf7466a 4f70e8b86d0ceb1e",
    "7680x4320/ff": "4bfaf1341a059fc0 9e6762b22b44a49b 1598c0a8594e7e66 32c30c2fd0384622 "
                    "3a30203e4e9ea094 73cf01dec0f9f3da 67177a11c33cad0b",
    "7680x4320/07": "e29fa4c64851bf08 2ab32b9e9e192885 5316b613cdce44dd a170b9177b0c5593 "
                    "b688d884c2384faa ad1bbf0b3866a1ba 0b7afbb60d37e9d7",
}


def make_cases(R: pyoracle.Reference, O: pyoracle.Oracle):
    rng = np.random.default_rng(20230501)
    cases, arrays = [], {}

    def add(name, img, taps=None, params=(1, 2, 6, 4), lanes=32, prefetch=True, expect=0):
        if taps is None:
            code, taps, msg = R.make_stream_taps(*params)
            assert code == 0, msg
        code, out, counters, msg = R.run_stream(img, taps, lanes=lanes, prefetch=prefetch)
        i = len(cases)
        arrays[f"img{i}"] = img
        meta = {"name": name, "w": int(img.shape[1]), "h": int(img.shape[0]),
                "taps": taps.as_dict(), "params": list(params), "lanes": lanes,
                "prefetch": bool(prefetch), "status": int(code), "message": msg}
        if code == 0:
            for k in PLANES:
                arrays[f"{k}{i}"] = out[k]
            arrays[f"u8{i}"] = O.clamp_abs(out["g"])
            meta["counters"] = counters
        else:
            assert code == expect, (name, code, msg)
        cases.append(meta)

    # SPEC / SURVEY Appendix A known answers
    ramp = np.tile(np.arange(5, dtype=np.uint8), (5, 1))
    add("ramp5", ramp)
    add("constant7", np.full((9, 11), 7, np.uint8))
    imp = np.zeros((9, 9), np.uint8)
    imp[4, 4] = 1
    add("impulse9", imp)
    step = np.zeros((5, 5), np.uint8)
    step[:, 3:] = 255
    add("step5", step)
    add("min5x5_random", rng.integers(0, 256, (5, 5), dtype=np.uint8))
    # ragged/odd sizes around the GPU warp (128 columns) and CTA (512) widths
    for (w, h) in [(6, 5), (5, 9), (37, 21), (64, 48), (131, 7), (132, 12), (133, 13),
                   (515, 9), (516, 11), (517, 6), (1029, 7)]:
        add(f"rand{w}x{h}", rng.integers(0, 256, (h, w), dtype=np.uint8),
            lanes=int(rng.choice([8, 16, 32, 64])), prefetch=bool(rng.integers(0, 2)))
    add("lowamp64x64", rng.integers(0, 256, (64, 64), dtype=np.uint8) & 7)
    # non-default parameter sets, including the wide_vagg regime
    for params in [(2, 2, 6, 4), (1, 3, 2, 1), (3, 1, 1, 1), (1, 64, 2, 3), (1, 32768, 1, 1),
                   (7, 5, 9, 11)]:
        code, taps, msg = R.make_stream_taps(*params)
        if code:
            continue
        add(f"params{params}", rng.integers(0, 256, (23, 70), dtype=np.uint8), taps=taps,
            params=params)
    # fault injection as in sobel5_cli.cpp:219 (even offset keeps parity)
    code, t, _ = R.make_stream_taps()
    t.k0[0] += 2
    add("fault_k0_plus2", rng.integers(0, 256, (32, 40), dtype=np.uint8), taps=t)
    # odd offset -> ParityViolation (pipeline.hpp:268-273)
    code, t, _ = R.make_stream_taps()
    t.k0[0] += 1
    add("fault_k0_plus1", rng.integers(0, 256, (16, 16), dtype=np.uint8), taps=t, expect=17)
    # ImageTooSmall
    add("too_small_4x9", np.zeros((9, 4), np.uint8), expect=13)
    return cases, arrays


def make_hashes(R: pyoracle.Reference, O: pyoracle.Oracle):
    out = {}
    code, taps, _ = R.make_stream_taps()
    for key, expect in SURVEY_A3.items():
        dims, mask = key.split("/")
        w, h = map(int, dims.split("x"))
        img = R.synth_random(w, h, 1) & int(mask, 16)
        code, o, counters, msg = R.run_stream(img, taps, lanes=256, prefetch=True,
                                              workers=os.cpu_count() or 1)
        assert code == 0, msg
        u8 = O.clamp_abs(o["g"])
        hs = [O.fnv1a64(img)] + [O.fnv1a64(o[k]) for k in PLANES] + [O.fnv1a64(u8)]
        got = " ".join(f"{x:016x}" for x in hs)
        assert got == expect, (key, got, expect)
        out[key] = {"w": w, "h": h, "mask": int(mask, 16), "seed": 1,
                    "fnv1a64": dict(zip(["input", *PLANES, "u8"], [f"{x:016x}" for x in hs])),
                    "sat255": float((u8 == 255).mean())}
        print(key, "ok", flush=True)
    return out


def make_known(R: pyoracle.Reference, O: pyoracle.Oracle):
    k = {}
    code, t, _ = R.make_stream_taps()
    k["default_taps"] = t.as_dict()
    k["taps"] = {}
    for params in [(2, 2, 6, 4), (1, 3, 2, 1), (1, 32768, 1, 1), (3, 1, 1, 1), (1, 1, 1, 1)]:
        code, t, msg = R.make_stream_taps(*params)
        k["taps"][str(params)] = t.as_dict() if code == 0 else {"error": code, "message": msg}
    k["errors"] = {}
    for params in [(0, (2, 1), (6, 1), (4, 1)), (1, (1, 2), (6, 1), (4, 1)),
                   (1, (0, 1), (6, 1), (4, 1)), (1, (2, 1), (-6, 1), (4, 1)),
                   (2, (1, 2), (6, 1), (4, 1)), (1, (65536, 1), (1, 1), (1, 1)),
                   (1, (200, 1), (200, 1), (1, 1)), (4, (1, 2), (1, 2), (1, 2))]:
        code, t, msg = R.make_stream_taps(*params)
        k["errors"][json.dumps(params)] = {"code": code, "message": msg,
                                           "taps": t.as_dict() if t else None}
    k["kernels"] = {}
    for params in [(1, 2, 6, 4), (2, 2, 6, 4), (1, 3, 2, 1)]:
        k["kernels"][str(params)] = [R.materialize(*params, d)[1].tolist() for d in range(4)]
    k["strips"] = {}
    for (w, lanes) in [(60, 32), (36, 32), (32, 32), (5, 8), (1024, 32), (7680, 256), (9, 5)]:
        code, strips, msg = R.plan_strips(w, lanes, 2)
        k["strips"][f"{w},{lanes}"] = {"code": code, "strips": strips, "message": msg}
    for (w, lanes, r) in [(10, 4, 2), (3, 32, 2), (10, 8, 0)]:
        code, strips, msg = R.plan_strips(w, lanes, r)
        k["strips"][f"{w},{lanes},{r}"] = {"code": code, "strips": strips, "message": msg}
    # counters at 1024^2 lanes 32 and a ragged plan, both modes
    k["counters"] = {}
    img = R.synth_random(1024, 1024, 1)
    for lanes, pf in [(32, True), (32, False)]:
        code, _, c, _ = R.run_stream(img, None, lanes=lanes, prefetch=pf, workers=8)
        k["counters"][f"1024x1024,{lanes},{int(pf)}"] = c
    img = R.synth_random(101, 37, 3)
    for lanes, pf in [(16, True), (64, False)]:
        code, _, c, _ = R.run_stream(img, None, lanes=lanes, prefetch=pf)
        k["counters"][f"101x37,{lanes},{int(pf)}"] = c
    # row helpers (pipeline.hpp:194-233, 268-273)
    rows = {"ramp": [1, 2, 3, 4, 5], "impulse": [0, 0, 1, 0, 0], "const7": [7] * 5,
            "d": [0, 1, 0, 3, 0], "long": list(range(10, 90, 7)), "short": [1, 2, 3, 4]}
    k["hpass"] = {}
    for name, row in rows.items():
        for which in range(5):
            code, out, msg = R.hpass(np.array(row, np.uint8), which)
            k["hpass"][f"{name},{which}"] = {"code": code, "out": out.tolist(), "message": msg}
    k["recover_diag"] = {}
    for s, d in [(10, 4), (0, 0), (3, 4), (-6, 2), (-7, 2)]:
        code, v, msg = R.recover_diag(s, d)
        k["recover_diag"][f"{s},{d}"] = {"code": code, "out": list(v), "message": msg}
    k["synth16"] = R.synth_random(16, 1, 1).ravel().tolist()
    return k


def main():
    if not pyoracle.ref_available():
        pyoracle.build()
    R, O = pyoracle.Reference(), pyoracle.Oracle()
    cases, arrays = make_cases(R, O)
    np.savez_compressed(os.path.join(HERE, "cases.npz"), **arrays)
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(cases, f, indent=1)
    with open(os.path.join(HERE, "known.json"), "w") as f:
        json.dump(make_known(R, O), f, indent=1)
    with open(os.path.join(HERE, "hashes.json"), "w") as f:
        json.dump(make_hashes(R, O), f, indent=1)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
