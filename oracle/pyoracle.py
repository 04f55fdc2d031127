"""ctypes bindings for the CPU oracle and the compiled reference.

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg import this module, and only as the
checker or the CPU timing arm.  The product (paper_2305_00515_b200) never
imports it.

* ``Oracle``  -> oracle/_build/libsobel5_oracle.so, the plain-C restatement
  (oracle/sobel5_oracle.c, every function citing the reference file:line).
* ``Reference`` -> oracle/_ref/libsobel5_ref.so, the reference's own headers
  compiled unmodified (oracle/Makefile, oracle/ref_shim.cpp).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libsobel5_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsobel5_ref.so")

TAP_FIELDS = ("f", "h", "k0", "k1", "gx_v", "gy_v", "gdm_f", "gdm_d")


class Taps(C.Structure):
    """POD mirror of sobel5::StreamTaps (pipeline.hpp:57-73)."""

    _fields_ = [("a", C.c_int32)] + [(n, C.c_int32 * 5) for n in TAP_FIELDS] + [
        ("wide_vagg", C.c_int32)
    ]

    def as_dict(self):
        d = {"a": self.a, "wide_vagg": self.wide_vagg}
        for n in TAP_FIELDS:
            d[n] = list(getattr(self, n))
        return d

    @classmethod
    def from_dict(cls, d):
        t = cls()
        t.a = d["a"]
        t.wide_vagg = int(d.get("wide_vagg", 0))
        for n in TAP_FIELDS:
            getattr(t, n)[:] = list(d[n])
        return t

    def copy(self):
        return Taps.from_dict(self.as_dict())


class Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "row_conv5_f", "row_conv5_h", "row_conv5_k0", "row_conv5_k1",
        "row_diff", "row_conv3_f", "row_conv3_h", "mac")]


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build():
    """Compile the oracle (and the reference shim where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _out_planes(w, h, want=True):
    ow, oh = w - 4, h - 4
    if not want:
        return None
    return {k: np.empty((oh, ow), np.int32) for k in ("gx", "gy", "gd", "gdt")} | {
        "g": np.empty((oh, ow), np.float64)}


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.oracle_make_stream_taps.argtypes = [C.c_int64] * 4 + [C.POINTER(Taps)]
        L.oracle_materialize.argtypes = [C.c_int64] * 4 + [C.c_int, C.c_void_p]
        L.oracle_run_stream.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(Taps)] + [
            C.c_void_p] * 7
        L.oracle_run_stream.restype = C.c_int
        L.oracle_sobel5_4d.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_int64] * 4 + [
            C.c_void_p] * 5
        L.oracle_sobel5_4d.restype = C.c_int
        L.oracle_clamp_abs_f64.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p]
        L.oracle_synth_random.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64]
        L.oracle_stream_counters.argtypes = [C.c_int, C.c_void_p, C.c_int, C.POINTER(Taps),
                                             C.c_int, C.POINTER(Counters)]
        L.oracle_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
        L.oracle_fnv1a64.restype = C.c_uint64
        L.oracle_pad_replicate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.oracle_pad_replicate.restype = C.c_int
        for fn in ("oracle_normalize_f64", "oracle_normalize_i32", "oracle_clamp_abs_i32"):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_size_t, C.c_void_p]
        L.oracle_conv2d_valid.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.oracle_conv2d_valid.restype = C.c_int
        L.oracle_conv2d_valid3.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.oracle_conv2d_valid3.restype = C.c_int
        L.oracle_sobel3_2d.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 3
        L.oracle_sobel3_2d.restype = C.c_int
        L.oracle_stream3_counters.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int,
                                              C.POINTER(Counters)]

    def make_stream_taps(self, a=1, b=2, m=6, n=4) -> Taps:
        t = Taps()
        self.lib.oracle_make_stream_taps(a, b, m, n, C.byref(t))
        return t

    def materialize(self, a, b, m, n, direction: int) -> np.ndarray:
        k = np.empty((5, 5), np.int32)
        self.lib.oracle_materialize(a, b, m, n, direction, _p(k))
        return k

    def run_stream(self, img: np.ndarray, taps: Taps | None = None):
        """Returns (status, planes dict, (bad_sum, bad_diff))."""
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        taps = taps or self.make_stream_taps()
        if w < 5 or h < 5:
            return 1, None, None
        o = _out_planes(w, h)
        bs, bd = np.zeros(1, np.int32), np.zeros(1, np.int32)
        st = self.lib.oracle_run_stream(_p(img), w, h, C.byref(taps), _p(o["gx"]), _p(o["gy"]),
                                        _p(o["gd"]), _p(o["gdt"]), _p(o["g"]), _p(bs), _p(bd))
        return st, o, (int(bs[0]), int(bd[0]))

    def sobel5_4d(self, img: np.ndarray, a=1, b=2, m=6, n=4):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        o = _out_planes(w, h)
        st = self.lib.oracle_sobel5_4d(_p(img), w, h, a, b, m, n, _p(o["gx"]), _p(o["gy"]),
                                       _p(o["gd"]), _p(o["gdt"]), _p(o["g"]))
        if st:
            raise RuntimeError(f"oracle_sobel5_4d status {st}")
        return o

    def conv2d_valid(self, img: np.ndarray, k: np.ndarray) -> np.ndarray:
        """oracle.hpp:19-49 for a 5x5 or 3x3 int32 kernel."""
        img = np.ascontiguousarray(img, np.uint8)
        k = np.ascontiguousarray(k, np.int32)
        ks = k.shape[0]
        h, w = img.shape
        out = np.empty((h - ks + 1, w - ks + 1), np.int32)
        fn = self.lib.oracle_conv2d_valid if ks == 5 else self.lib.oracle_conv2d_valid3
        if fn(_p(img), w, h, _p(k), _p(out)):
            raise ValueError("image smaller than the kernel")
        return out

    def clamp_abs(self, g: np.ndarray) -> np.ndarray:
        g = np.ascontiguousarray(g, np.float64)
        out = np.empty(g.shape, np.uint8)
        self.lib.oracle_clamp_abs_f64(_p(g), g.size, _p(out))
        return out

    def synth_random(self, w, h, seed=1) -> np.ndarray:
        img = np.empty((h, w), np.uint8)
        self.lib.oracle_synth_random(_p(img), w, h, seed)
        return img

    def stream_counters(self, h, strip_widths, taps: Taps | None = None, prefetch=True):
        taps = taps or self.make_stream_taps()
        sw = np.ascontiguousarray(strip_widths, np.int32)
        c = Counters()
        self.lib.oracle_stream_counters(h, _p(sw), len(sw), C.byref(taps), int(prefetch),
                                        C.byref(c))
        return {n: getattr(c, n) for n, _ in Counters._fields_}

    def fnv1a64(self, a: np.ndarray) -> int:
        a = np.ascontiguousarray(a)
        return int(self.lib.oracle_fnv1a64(_p(a), a.nbytes))

    # ---- detect path ----
    def pad_replicate(self, img: np.ndarray, r: int = 2):
        """Returns (status, padded) -- status 0, 20 EmptyPlane, 19 DimMismatch."""
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        out = np.empty((max(h + 2 * r, 0), max(w + 2 * r, 0)), np.uint8)
        st = self.lib.oracle_pad_replicate(_p(img), w, h, r, _p(out))
        return st, (out if st == 0 else None)

    def quantize(self, plane: np.ndarray, mode: str) -> np.ndarray:
        """detail::quantize of a RealPlane (float64) or SignedPlane (int32)."""
        out = np.empty(plane.shape, np.uint8)
        if plane.dtype == np.float64:
            plane = np.ascontiguousarray(plane)
            if mode == "clamp_abs":
                self.lib.oracle_clamp_abs_f64(_p(plane), plane.size, _p(out))
            else:
                self.lib.oracle_normalize_f64(_p(plane), plane.size, _p(out))
        else:
            plane = np.ascontiguousarray(plane, np.int32)
            fn = "oracle_clamp_abs_i32" if mode == "clamp_abs" else "oracle_normalize_i32"
            getattr(self.lib, fn)(_p(plane), plane.size, _p(out))
        return out

    def sobel3_2d(self, img: np.ndarray):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        if w < 3 or h < 3:
            return 1, None
        o = {k: np.empty((h - 2, w - 2), np.int32) for k in ("gx", "gy")}
        o["g"] = np.empty((h - 2, w - 2), np.float64)
        st = self.lib.oracle_sobel3_2d(_p(img), w, h, _p(o["gx"]), _p(o["gy"]), _p(o["g"]))
        return st, o

    def stream3_counters(self, h, strip_widths, prefetch=True):
        sw = np.ascontiguousarray(strip_widths, np.int32)
        c = Counters()
        self.lib.oracle_stream3_counters(h, _p(sw), len(sw), int(prefetch), C.byref(c))
        return {n: getattr(c, n) for n, _ in Counters._fields_}


class Reference:
    """The reference's own headers, compiled (oracle/_ref/libsobel5_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        E = [C.c_char_p, C.c_int]
        L.ref_make_stream_taps.argtypes = [C.c_int64] * 7 + [C.POINTER(Taps)] + E
        L.ref_materialize.argtypes = [C.c_int64] * 4 + [C.c_int, C.c_void_p] + E
        L.ref_run_stream.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(Taps), C.c_int,
                                     C.c_int, C.c_int] + [C.c_void_p] * 6 + E
        L.ref_sobel5_4d.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_int64] * 4 + [
            C.c_void_p] * 5 + E
        L.ref_diag_via_sum_diff.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                            C.c_void_p] + E
        L.ref_synth_random.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64]
        L.ref_plan_strips.argtypes = [C.c_int] * 4 + [C.c_void_p] * 4 + E
        L.ref_hpass.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_int64] * 4 + [
            C.c_void_p] + E
        L.ref_recover_diag.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p] + E
        L.ref_measure_run_stream.argtypes = [C.c_void_p] + [C.c_int] * 6 + [C.c_void_p]
        L.ref_measure_run_stream.restype = C.c_double
        L.ref_measure_oracle.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.ref_measure_oracle.restype = C.c_double
        L.ref_pad_replicate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p] + E
        L.ref_quantize.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.ref_sobel3_2d.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 3 + E
        L.ref_run_stream_3x3.argtypes = [C.c_void_p] + [C.c_int] * 5 + [C.c_void_p] * 4 + E
        L.ref_measure_run_stream_3x3.argtypes = [C.c_void_p] + [C.c_int] * 6 + [C.c_void_p]
        L.ref_measure_run_stream_3x3.restype = C.c_double
        L.ref_conv2d_valid.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                       C.c_void_p]
        L.ref_conv2d_valid.restype = C.c_int
        L.ref_measure_csv.argtypes = [C.c_void_p] + [C.c_int] * 7 + [C.c_void_p]
        L.ref_measure_csv.restype = C.c_double

    @staticmethod
    def _err():
        return C.create_string_buffer(512)

    def make_stream_taps(self, a=1, b=(2, 1), m=(6, 1), n=(4, 1)):
        """Returns (code, Taps | None, message). Rationals as (num, den)."""
        b, m, n = [(x, 1) if isinstance(x, int) else x for x in (b, m, n)]
        t, e = Taps(), self._err()
        code = self.lib.ref_make_stream_taps(a, b[0], b[1], m[0], m[1], n[0], n[1], C.byref(t),
                                             e, 512)
        return code, (t if code == 0 else None), e.value.decode()

    def materialize(self, a, b, m, n, direction):
        k, e = np.empty((5, 5), np.int32), self._err()
        code = self.lib.ref_materialize(a, b, m, n, direction, _p(k), e, 512)
        return code, k, e.value.decode()

    def run_stream(self, img, taps: Taps | None = None, lanes=32, prefetch=True, workers=1):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        if taps is None:
            taps = self.make_stream_taps()[1]
        o = _out_planes(max(w, 5), max(h, 5))
        cnt = np.zeros(8, np.uint64)
        e = self._err()
        code = self.lib.ref_run_stream(_p(img), w, h, C.byref(taps), lanes, int(prefetch),
                                       workers, _p(o["gx"]), _p(o["gy"]), _p(o["gd"]),
                                       _p(o["gdt"]), _p(o["g"]), _p(cnt), e, 512)
        names = [n for n, _ in Counters._fields_]
        return code, o, dict(zip(names, (int(x) for x in cnt))), e.value.decode()

    def sobel5_4d(self, img, a=1, b=2, m=6, n=4):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        o = _out_planes(w, h)
        e = self._err()
        code = self.lib.ref_sobel5_4d(_p(img), w, h, a, b, m, n, _p(o["gx"]), _p(o["gy"]),
                                      _p(o["gd"]), _p(o["gdt"]), _p(o["g"]), e, 512)
        if code:
            raise RuntimeError(e.value.decode())
        return o

    def diag_via_sum_diff(self, img):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        gd, gdt = np.empty((h - 4, w - 4), np.int32), np.empty((h - 4, w - 4), np.int32)
        e = self._err()
        code = self.lib.ref_diag_via_sum_diff(_p(img), w, h, _p(gd), _p(gdt), e, 512)
        return code, gd, gdt

    def synth_random(self, w, h, seed=1):
        img = np.empty((h, w), np.uint8)
        self.lib.ref_synth_random(_p(img), w, h, seed)
        return img

    def plan_strips(self, width, lanes, radius=2):
        cap = max(1, width + 1)
        bufs = [np.zeros(cap, np.int32) for _ in range(3)]
        n = C.c_int(0)
        e = self._err()
        code = self.lib.ref_plan_strips(width, lanes, radius, cap, C.byref(n), *map(_p, bufs), e,
                                        512)
        if code:
            return code, None, e.value.decode()
        k = n.value
        return 0, [(int(bufs[0][i]), int(bufs[1][i]), int(bufs[2][i])) for i in range(k)], ""

    def hpass(self, row, which, a=1, b=2, m=6, n=4):
        row = np.ascontiguousarray(row, np.uint8)
        out = np.zeros(max(1, row.size - 4), np.int32)
        e = self._err()
        code = self.lib.ref_hpass(_p(row), row.size, which, a, b, m, n, _p(out), e, 512)
        return code, out[: max(0, row.size - 4)], e.value.decode()

    def recover_diag(self, s, d):
        gd, gdt = np.zeros(1, np.int32), np.zeros(1, np.int32)
        e = self._err()
        code = self.lib.ref_recover_diag(s, d, _p(gd), _p(gdt), e, 512)
        return code, (int(gd[0]), int(gdt[0])), e.value.decode()

    def measure_run_stream(self, img, lanes=256, prefetch=True, workers=1, iters=1):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        sd = np.zeros(1, np.float64)
        mean = self.lib.ref_measure_run_stream(_p(img), w, h, lanes, int(prefetch), workers,
                                               iters, _p(sd))
        return mean, float(sd[0])


    # ---- detect path ----
    def pad_replicate(self, img, r=2):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape if img.size else (0, 0)
        out = np.empty((max(h + 2 * r, 0), max(w + 2 * r, 0)), np.uint8)
        e = self._err()
        code = self.lib.ref_pad_replicate(_p(img), w, h, r, _p(out), e, 512)
        return code, (out if code == 0 else None), e.value.decode()

    def quantize(self, plane, mode):
        out = np.empty(plane.shape, np.uint8)
        kind = 0 if plane.dtype == np.float64 else 1
        plane = np.ascontiguousarray(plane, np.float64 if kind == 0 else np.int32)
        h, w = plane.shape
        self.lib.ref_quantize(_p(plane), kind, w, h, 1 if mode == "normalize" else 0, _p(out))
        return out

    def conv2d_valid(self, img, k):
        img = np.ascontiguousarray(img, np.uint8)
        k = np.ascontiguousarray(k, np.int32)
        ks = k.shape[0]
        h, w = img.shape
        out = np.empty((max(h - ks + 1, 0), max(w - ks + 1, 0)), np.int32)
        st = self.lib.ref_conv2d_valid(_p(img), w, h, _p(k), ks, _p(out))
        return st, out

    def sobel3_2d(self, img):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        o = {k: np.empty((max(h - 2, 1), max(w - 2, 1)), np.int32) for k in ("gx", "gy")}
        o["g"] = np.empty((max(h - 2, 1), max(w - 2, 1)), np.float64)
        e = self._err()
        code = self.lib.ref_sobel3_2d(_p(img), w, h, _p(o["gx"]), _p(o["gy"]), _p(o["g"]), e, 512)
        return code, o, e.value.decode()

    def run_stream_3x3(self, img, lanes=32, prefetch=True, workers=1):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        o = {k: np.empty((max(h - 2, 1), max(w - 2, 1)), np.int32) for k in ("gx", "gy")}
        o["g"] = np.empty((max(h - 2, 1), max(w - 2, 1)), np.float64)
        cnt = np.zeros(8, np.uint64)
        e = self._err()
        code = self.lib.ref_run_stream_3x3(_p(img), w, h, lanes, int(prefetch), workers,
                                           _p(o["gx"]), _p(o["gy"]), _p(o["g"]), _p(cnt), e, 512)
        names = [n for n, _ in Counters._fields_]
        return code, o, dict(zip(names, (int(x) for x in cnt))), e.value.decode()

    def measure_csv(self, img, which="fast", lanes=32, prefetch=True, workers=1, iters=1):
        """(mean_s, csv_row) of the reference's measure() around run_stream
        (which="fast") or the sobel5_4d oracle (which="oracle"); the row in
        the reference's BenchReport CSV schema and number format
        (metrics.hpp:129-139: setprecision 9 for the times, 6 for the rates)."""
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        f = np.zeros(4, np.float64)
        mean = self.lib.ref_measure_csv(_p(img), w, h, 0 if which == "fast" else 1, lanes,
                                        int(prefetch), workers, iters, _p(f))
        label = "fast-5x5" if which == "fast" else "oracle-5x5"
        row = f"{label},{w},{h},{iters},{f[0]:.9g},{f[1]:.9g},{f[2]:.6g},{f[3]:.6g}"
        return mean, row

    def measure_run_stream_3x3(self, img, lanes=256, prefetch=True, workers=1, iters=1):
        img = np.ascontiguousarray(img, np.uint8)
        h, w = img.shape
        sd = np.zeros(1, np.float64)
        mean = self.lib.ref_measure_run_stream_3x3(_p(img), w, h, lanes, int(prefetch), workers,
                                                   iters, _p(sd))
        return mean, float(sd[0])


def ref_available() -> bool:
    return os.path.exists(REF_SO)
