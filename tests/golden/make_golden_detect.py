"""Golden fixtures of the detect path and the 3x3 path, from the REFERENCE.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden_detect.py

Every output comes from oracle/_ref/libsobel5_ref.so, the reference headers
compiled unmodified: pad_replicate and detail::quantize (image_io.hpp,
compiled against the declaration-only oracle/png_stub/png.h), run_stream
(pipeline.hpp), run_stream_3x3 (pipeline.hpp:551-573) and sobel3_2d
(oracle.hpp:58-70).

Outputs:
  detect.npz   <case>__img, <case>__clamp_abs, <case>__normalize: the CLI
               detect flow (sobel5_cli.cpp:127-177) with --pad replicate:
               quantize(run_stream(pad_replicate(img, 2).plane).g, mode)
  sobel3.npz   <case>__img, __gx, __gy, __g from run_stream_3x3 (lanes 32,
               prefetch on) -- equal to sobel3_2d, which is checked here too
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle  # noqa: E402


def images(R):
    rng = np.random.default_rng(2305)
    out = {
        "rand64x48": rng.integers(0, 256, (48, 64), dtype=np.uint8),
        "low97x61": R.synth_random(97, 61, 7) & 0x07,
        "tiny5x3": rng.integers(0, 256, (3, 5), dtype=np.uint8),
        "one1x1": np.array([[200]], np.uint8),
        "step150x40": np.where(np.arange(150)[None, :] >= 70, 255, 0).astype(np.uint8).repeat(
            40, 0),
        "mask0f_200x131": R.synth_random(200, 131, 3) & 0x0F,
        "ramp131x9": (np.arange(131, dtype=np.int64)[None, :] * 2 % 256).astype(np.uint8).repeat(
            9, 0),
        "wide520x7": R.synth_random(520, 7, 11) & 0x3F,
    }
    return {k: np.ascontiguousarray(v, np.uint8) for k, v in out.items()}


def main():
    R = pyoracle.Reference()
    det, s3 = {}, {}
    taps = R.make_stream_taps()[1]
    for name, img in images(R).items():
        code, padded, msg = R.pad_replicate(img, 2)
        assert code == 0, msg
        code, planes, _, msg = R.run_stream(padded, taps, lanes=32, prefetch=True)
        assert code == 0, msg
        det[f"{name}__img"] = img
        for mode in ("clamp_abs", "normalize"):
            det[f"{name}__{mode}"] = R.quantize(planes["g"], mode)
        h, w = img.shape
        if w >= 3 and h >= 3:
            code, o, _, msg = R.run_stream_3x3(img, lanes=32, prefetch=True)
            assert code == 0, msg
            code2, o2, msg2 = R.sobel3_2d(img)
            assert code2 == 0, msg2
            for k in ("gx", "gy", "g"):
                assert np.array_equal(o[k], o2[k]), (name, k)
                s3[f"{name}__{k}"] = o[k]
            s3[f"{name}__img"] = img
    np.savez_compressed(os.path.join(HERE, "detect.npz"), **det)
    np.savez_compressed(os.path.join(HERE, "sobel3.npz"), **s3)
    print(f"detect.npz: {len(det) // 3} cases, sobel3.npz: {len(s3) // 4} cases")


if __name__ == "__main__":
    main()
