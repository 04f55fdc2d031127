"""Python mirror of the reference's run_stream interface over the C ABI.

Names, argument meaning and error behaviour follow the reference headers
(proj/include/sobel5/): ``FilterParams``/``validate_params``/``materialize``
(filter_algebra.hpp:58-199), ``make_stream_taps`` (pipeline.hpp:75-107),
``plan_strips`` (strips.hpp:35-61), ``Prefetch`` (pipeline.hpp:21),
``StreamResult`` (pipeline.hpp:284-291) and ``run_stream``
(pipeline.hpp:452-477).  The compute always runs on the GPU through
libsobel5_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import sys
import threading
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _abi
from ._abi import Counters, Diag, Planes, Taps

# ---- errors (reference errors.hpp:9-32) -------------------------------------


class Error(RuntimeError):
    pass


class NonPositiveParam(Error): pass
class NonIntegralWeight(Error): pass
class ParamOverflow(Error): pass
class ImageTooSmall(Error): pass
class RowTooShort(Error): pass
class MissingRow(Error): pass
class VariantMismatch(Error): pass
class ParityViolation(Error): pass
class LaneTooNarrow(Error): pass
class DimMismatch(Error): pass
class EmptyPlane(Error): pass
class CudaError(Error): pass


_STATUS_EXC = {
    _abi.EMPTY_PLANE: EmptyPlane,
    _abi.IMAGE_TOO_SMALL: ImageTooSmall,
    _abi.DIM_MISMATCH: DimMismatch,
    _abi.PARITY_VIOLATION: ParityViolation,
    _abi.NON_POSITIVE_PARAM: NonPositiveParam,
    _abi.PARAM_OVERFLOW: ParamOverflow,
    _abi.LANE_TOO_NARROW: LaneTooNarrow,
}


def check(status: int, what: str = "") -> None:
    if status == _abi.OK:
        return
    exc = _STATUS_EXC.get(status, CudaError)
    msg = _abi.status_string(status)
    raise exc(f"{what}: {msg}" if what else msg)


# ---- filter algebra (filter_algebra.hpp) ------------------------------------

K_MAX_WEIGHT_MAGNITUDE = 1 << 15  # filter_algebra.hpp:148
DIRECTIONS = ("Kx", "Ky", "Kd", "Kdt")  # direction_name, filter_algebra.hpp:67-75


def _rat_str(r: Fraction) -> str:
    return str(r.numerator) if r.denominator == 1 else f"{r.numerator}/{r.denominator}"


@dataclass(frozen=True)
class FilterParams:
    """(a, b, m, n) of Eq. 5; defaults reproduce Eq. 3 (filter_algebra.hpp:58-63)."""

    a: int = 1
    b: Fraction | int = 2
    m: Fraction | int = 6
    n: Fraction | int = 4


def _materialize_exact(p: FilterParams, direction: int):
    """filter_algebra.hpp:82-134 (exact rationals)."""
    a, b, m, n = Fraction(p.a), Fraction(p.b), Fraction(p.m), Fraction(p.n)
    one, zero = Fraction(1), Fraction(0)
    if direction == 0:
        col, row = (one, n, m, n, one), (-one, -b, zero, b, one)
        return [[a * col[i] * row[j] for j in range(5)] for i in range(5)]
    if direction == 1:
        col, row = (-one, -b, zero, b, one), (one, n, m, n, one)
        return [[a * col[i] * row[j] for j in range(5)] for i in range(5)]
    nb, mb = n * b, m * b
    if direction == 2:
        k = [[-m, -n, -one, -b, zero], [-n, -mb, -nb, zero, b], [-one, -nb, zero, nb, one],
             [-b, zero, nb, mb, n], [zero, b, one, n, m]]
    else:
        k = [[zero, -b, -one, -n, -m], [b, zero, -nb, -mb, -n], [one, nb, zero, -nb, -one],
             [n, mb, nb, zero, -b], [m, n, one, b, zero]]
    return [[a * e for e in row] for row in k]


def validate_params(p: FilterParams) -> None:
    """filter_algebra.hpp:157-188, same checks, order and messages."""
    if p.a < 1:
        raise NonPositiveParam(f"a = {p.a} must be a positive integer")
    for name in ("b", "m", "n"):
        v = Fraction(getattr(p, name))
        if v <= 0:
            raise NonPositiveParam(f"{name} = {_rat_str(v)} must be positive")
    max_mag = 0
    for d in range(4):
        k = _materialize_exact(p, d)
        for i in range(5):
            for j in range(5):
                if k[i][j].denominator != 1:
                    raise NonIntegralWeight(
                        f"{DIRECTIONS[d]}({i},{j}) = {_rat_str(k[i][j])} is not an integer")
                max_mag = max(max_mag, abs(k[i][j].numerator))
    for name in ("b", "m", "n"):
        v = Fraction(getattr(p, name))
        if v.denominator != 1:
            raise NonIntegralWeight(f"parameter {name} = {_rat_str(v)} must be an integer "
                                    "(streaming taps are integer vectors)")
    if max_mag > K_MAX_WEIGHT_MAGNITUDE:
        raise ParamOverflow(f"largest weight magnitude {max_mag} exceeds "
                            f"{K_MAX_WEIGHT_MAGNITUDE}")


def materialize(p: FilterParams, direction: int) -> np.ndarray:
    """filter_algebra.hpp:192-199 (params must already be valid)."""
    k = _materialize_exact(p, direction)
    return np.array([[int(e) for e in row] for row in k], dtype=np.int32)


KERNELS = ("packed_default", "packed_runtime_taps", "f32x2_runtime_taps", "generic")


def kernel_for(taps: Taps) -> str:
    """Kernel family the C ABI selects for these taps (sobel5_kernel_for_taps)."""
    return KERNELS[_abi.load().sobel5_kernel_for_taps(C.byref(taps))]


def make_stream_taps(p: FilterParams = FilterParams()) -> Taps:
    """pipeline.hpp:75-107 (validation, then the C ABI builds the taps)."""
    validate_params(p)
    t = Taps()
    check(_abi.load().sobel5_make_taps(int(p.a), int(Fraction(p.b)), int(Fraction(p.m)),
                                       int(Fraction(p.n)), C.byref(t)), "make_stream_taps")
    return t


# ---- strips (strips.hpp) ------------------------------------------------------


@dataclass(frozen=True)
class Strip:
    in_off: int = 0
    out_off: int = 0
    out_w: int = 0


@dataclass
class StripPlan:
    in_width: int = 0
    out_width: int = 0
    lane_width: int = 0
    radius: int = 0
    strips: list = field(default_factory=list)


def plan_strips(width: int, lane_width: int, radius: int) -> StripPlan:
    """strips.hpp:35-61, same errors and messages."""
    if radius <= 0:
        raise DimMismatch(f"strip radius must be positive, got {radius}")
    if lane_width <= 2 * radius:
        raise LaneTooNarrow(f"lane width {lane_width} leaves no output columns at radius "
                            f"{radius}")
    if width < 2 * radius + 1:
        raise ImageTooSmall(f"width {width} is below the minimum {2 * radius + 1} for radius "
                            f"{radius}")
    plan = StripPlan(width, width - 2 * radius, lane_width, radius, [])
    step = lane_width - 2 * radius
    for off in range(0, plan.out_width, step):
        plan.strips.append(Strip(off, off, min(step, plan.out_width - off)))
    return plan


# ---- run_stream -----------------------------------------------------------------


class Prefetch(enum.IntEnum):
    off = 0
    on = 1


@dataclass
class StreamResult:
    gx: np.ndarray
    gy: np.ndarray
    gd: np.ndarray
    gdt: np.ndarray
    g: np.ndarray
    counters: dict
    u8: np.ndarray | None = None


def plan_counters(height: int, plan: StripPlan, taps: Taps, prefetch: Prefetch) -> dict:
    """Reference-schedule OpCounters (pipeline.hpp:26-51, closed form)."""
    widths = np.array([s.out_w for s in plan.strips], dtype=np.int32)
    c = Counters()
    check(_abi.load().sobel5_plan_counters(height, widths.ctypes.data_as(C.c_void_p),
                                           len(widths), C.byref(taps), int(prefetch),
                                           C.byref(c)), "plan_counters")
    return {n: int(getattr(c, n)) for n, _ in Counters._fields_}


class Context:
    """Per-thread, per-device context (streams + cached device buffers)."""

    def __init__(self, device: int = 0):
        self._lib = _abi.load()
        h = C.c_void_p()
        check(self._lib.sobel5_ctx_create(C.byref(h), device), "sobel5_ctx_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.sobel5_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def last_error(self) -> str:
        return self._lib.sobel5_ctx_last_error(self._h).decode()

    def run_host(self, img: np.ndarray, taps: Taps, prefetch: Prefetch = Prefetch.on,
                 planes=("gx", "gy", "gd", "gdt", "g"), out: dict | None = None):
        """Host arrays in / out.  Returns (status, dict of planes, Diag)."""
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape
        ow, oh = max(w - 4, 0), max(h - 4, 0)
        dt = {"gx": np.int32, "gy": np.int32, "gd": np.int32, "gdt": np.int32, "g": np.float64,
              "g32": np.float32, "u8": np.uint8}
        res = out if out is not None else {
            k: np.empty((oh, ow), dt[k]) for k in planes} if (ow > 0 and oh > 0) else {}
        pl = Planes(pitch=ow)
        for k, v in res.items():
            setattr(pl, k, v.ctypes.data)
        d = Diag()
        st = self._lib.sobel5_run_host(self._h, img.ctypes.data, w, h, C.byref(taps),
                                       int(prefetch), C.byref(pl), C.byref(d))
        return st, res, d


    def run_host_frames(self, frames: np.ndarray, taps: Taps, prefetch: Prefetch = Prefetch.on,
                        planes=("gx", "gy", "gd", "gdt", "g"), out: dict | None = None):
        """sobel5_run_host_frames: a stream of frames (n, h, w) uint8 end to
        end, run_stream per frame, pipelined across frames.  Returns
        (status, dict of (n, h - 4, w - 4) planes, Diag)."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        n, h, w = frames.shape
        ow, oh = max(w - 4, 0), max(h - 4, 0)
        dt = {"gx": np.int32, "gy": np.int32, "gd": np.int32, "gdt": np.int32, "g": np.float64,
              "g32": np.float32, "u8": np.uint8}
        res = out if out is not None else {
            k: np.empty((n, oh, ow), dt[k]) for k in planes} if (ow > 0 and oh > 0) else {}
        pl = Planes(pitch=ow)
        for k, v in res.items():
            setattr(pl, k, v.ctypes.data)
        d = Diag()
        st = self._lib.sobel5_run_host_frames(self._h, frames.ctypes.data, w, h, n, w * h,
                                              C.byref(taps), int(prefetch), C.byref(pl), ow * oh,
                                              C.byref(d))
        return st, res, d

    def detect_host(self, img: np.ndarray, taps: Taps, prefetch: Prefetch = Prefetch.on,
                    pad: bool = True, save_mode: "SaveMode" = None, planes=()):
        """sobel5_detect_host: returns (status, u8 edge map, dict of planes, Diag)."""
        save_mode = SaveMode.normalize if save_mode is None else save_mode
        img = np.ascontiguousarray(img, dtype=np.uint8)
        h, w = img.shape if img.ndim == 2 else (0, 0)
        ow, oh = (w, h) if pad else (max(w - 4, 0), max(h - 4, 0))
        dt = {"gx": np.int32, "gy": np.int32, "gd": np.int32, "gdt": np.int32, "g": np.float64,
              "g32": np.float32}
        u8 = np.empty((oh, ow), np.uint8)
        res = {k: np.empty((oh, ow), dt[k]) for k in planes}
        pl = Planes(pitch=ow)
        for k, v in res.items():
            setattr(pl, k, v.ctypes.data)
        d = Diag()
        st = self._lib.sobel5_detect_host(self._h, img.ctypes.data if img.size else None, w, h,
                                          C.byref(taps), int(prefetch), int(bool(pad)),
                                          int(save_mode), u8.ctypes.data if u8.size else None,
                                          C.byref(pl) if planes else None, C.byref(d))
        return st, u8, res, d


_tls = threading.local()


def _current_device() -> int:
    """The caller's current CUDA device (torch's, when torch is in use)."""
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_available():
        return torch.cuda.current_device()
    return 0


def default_context(device: int | None = None) -> Context:
    """One context per host thread and device, like the C++ mirror's
    gpu::thread_context() (include/sobel5_b200/stream.hpp): a sobel5_ctx is
    not thread-safe (pinned staging, streams, the pending split call), and
    ctypes releases the GIL during the C call, so threads must not share
    one.  The reference's run_stream is reentrant (pipeline.hpp:452)."""
    dev = _current_device() if device is None else device
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    ctx = ctxs.get(dev)
    if ctx is None:
        ctx = ctxs[dev] = Context(dev)
    return ctx


def run_stream(img: np.ndarray, taps_or_params, plan: StripPlan, prefetch: Prefetch,
               workers: int = 1, ctx: Context | None = None) -> StreamResult:
    """Drop-in for sobel5::run_stream (pipeline.hpp:452-477).

    ``workers`` is accepted and ignored (the GPU grid replaces the thread
    pool); ``plan`` is validated like the reference and drives the
    reference-schedule counters, while the GPU tiling is independent of it
    (SPEC.md: correctness is independent of the plan).
    """
    img = np.ascontiguousarray(img, dtype=np.uint8)
    if img.ndim != 2:
        raise DimMismatch("image must be 2-D")
    h, w = img.shape
    if w < 5 or h < 5:  # pipeline.hpp:454-456
        raise ImageTooSmall(f"streaming filter needs at least 5x5, got {w}x{h}")
    if plan.in_width != w or plan.radius != 2:  # pipeline.hpp:457-460
        raise DimMismatch(f"strip plan covers {plan.in_width} columns at radius {plan.radius}, "
                          f"image has {w}")
    taps = taps_or_params if isinstance(taps_or_params, Taps) else make_stream_taps(
        taps_or_params)
    ctx = ctx or default_context()
    # the plan orders the reported ParityViolation pair (strip-major, as the
    # reference with workers = 1)
    check(_abi.load().sobel5_ctx_set_strip_width(ctx.handle, plan.lane_width - 2 * plan.radius),
          "sobel5_ctx_set_strip_width")
    st, res, d = ctx.run_host(img, taps, prefetch)
    if st == _abi.PARITY_VIOLATION:  # pipeline.hpp:269-271
        raise ParityViolation(f"odd sum/difference pair ({d.sum}, {d.diff})")
    if st != _abi.OK:
        check(st, f"run_stream ({ctx.last_error()})")
    return StreamResult(res["gx"], res["gy"], res["gd"], res["gdt"], res["g"],
                        plan_counters(h, plan, taps, prefetch))


def conv2d_valid(img: np.ndarray, kernel, ctx: Context | None = None) -> np.ndarray:
    """oracle.hpp:19-49 on the GPU (sobel5_conv2d_valid_host): valid-mode
    correlation with a 5x5 or 3x3 integer kernel, int32 result."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    k = np.ascontiguousarray(kernel, dtype=np.int32)
    if k.ndim != 2 or k.shape[0] != k.shape[1] or k.shape[0] not in (3, 5):
        raise DimMismatch("kernel must be 5x5 or 3x3")
    ks = k.shape[0]
    h, w = img.shape
    if w < ks or h < ks:
        raise ImageTooSmall(f"conv2d_valid needs at least {ks}x{ks}, got {w}x{h}")
    out = np.empty((h - ks + 1, w - ks + 1), np.int32)
    ctx = ctx or default_context()
    check(_abi.load().sobel5_conv2d_valid_host(ctx.handle, img.ctypes.data, w, h, k.ctypes.data, ks,
                                               out.ctypes.data), "conv2d_valid")
    return out


def sobel5_4d(img: np.ndarray, params: FilterParams = FilterParams(),
              ctx: Context | None = None) -> StreamResult:
    """oracle.hpp:82-98: the four dense correlations with the materialised
    kernels plus the double magnitude, on the GPU (sobel5_dense_4d_host) --
    the oracle's algorithm, independent of run_stream's streaming kernels.
    counters are empty (the oracle keeps none)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    if w < 5 or h < 5:
        raise ImageTooSmall(f"conv2d_valid needs at least 5x5, got {w}x{h}")
    validate_params(params)
    k = np.ascontiguousarray(np.stack([materialize(params, d) for d in range(4)]), np.int32)
    ow, oh = w - 4, h - 4
    res = {n: np.empty((oh, ow), np.int32) for n in ("gx", "gy", "gd", "gdt")}
    res["g"] = np.empty((oh, ow), np.float64)
    pl = Planes(pitch=ow)
    for n, v in res.items():
        setattr(pl, n, v.ctypes.data)
    ctx = ctx or default_context()
    check(_abi.load().sobel5_dense_4d_host(ctx.handle, img.ctypes.data, w, h, k.ctypes.data,
                                           C.byref(pl)), "sobel5_4d")
    return StreamResult(res["gx"], res["gy"], res["gd"], res["gdt"], res["g"], {})


def diag_via_sum_diff(img: np.ndarray, params: FilterParams = FilterParams()):
    """oracle.hpp:100-129: (gd, gdt) through the Kd+/- sum and difference
    kernels, equal to run_stream's diagonals for valid params (GPU)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    if w < 5 or h < 5:
        raise ImageTooSmall(f"conv2d_valid needs at least 5x5, got {w}x{h}")
    st, res, d = default_context().run_host(img, make_stream_taps(params), Prefetch.on,
                                            planes=("gd", "gdt"))
    check(st, "diag_via_sum_diff")
    return res["gd"], res["gdt"]


def synth_random(width: int, height: int, seed: int) -> np.ndarray:
    """synth.hpp:20-35 on the host: pixel i is byte (i mod 8) of the
    splitmix64 output word floor(i / 8) (vectorised random-access form)."""
    n = width * height
    k = np.arange((n + 7) // 8, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (k + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z.view(np.uint8)[:n].reshape(height, width).copy()


# ---- device-resident helpers (torch tensors as device memory) --------------------


def round_up(v: int, m: int) -> int:
    return (v + m - 1) // m * m


def alloc_input(width: int, height: int, device="cuda", frames: int = 1):
    """Pitched uint8 device image(s): returns (tensor, pitch_bytes)."""
    import torch
    pitch = round_up(width, 128)
    t = torch.empty((frames, height, pitch) if frames > 1 else (height, pitch),
                    dtype=torch.uint8, device=device)
    return t, pitch


def alloc_planes(out_w: int, out_h: int, which=("gx", "gy", "gd", "gdt", "g"), device="cuda",
                 frames: int = 1):
    """Pitched device planes sharing one element pitch: (dict, pitch_elems)."""
    import torch
    pitch = round_up(out_w, 32)
    dt = {"gx": torch.int32, "gy": torch.int32, "gd": torch.int32, "gdt": torch.int32,
          "g": torch.float64, "g32": torch.float32, "u8": torch.uint8}
    shape = (frames, out_h, pitch) if frames > 1 else (out_h, pitch)
    return {k: torch.empty(shape, dtype=dt[k], device=device) for k in which}, pitch


def planes_struct(planes: dict, pitch: int) -> Planes:
    pl = Planes(pitch=pitch)
    for k, v in planes.items():
        setattr(pl, k, v.data_ptr())
    return pl


def launch(d_in, in_pitch: int, width: int, height: int, taps: Taps, prefetch: int,
           planes: dict, pitch: int, diag=None, stream=None) -> None:
    """Enqueue one device-resident image (sobel5_launch)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    pl = planes_struct(planes, pitch)
    check(_abi.load().sobel5_launch(d_in.data_ptr(), in_pitch, width, height, C.byref(taps),
                                    int(prefetch), C.byref(pl),
                                    None if diag is None else diag.data_ptr(), s),
          "sobel5_launch")


def launch_batch(d_in, in_pitch: int, in_frame_stride: int, width: int, height: int,
                 n_frames: int, taps: Taps, prefetch: int, planes: dict, pitch: int,
                 out_frame_stride: int, diag=None, stream=None) -> None:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    pl = planes_struct(planes, pitch)
    check(_abi.load().sobel5_launch_batch(d_in.data_ptr(), in_pitch, in_frame_stride, width,
                                          height, n_frames, C.byref(taps), int(prefetch),
                                          C.byref(pl), out_frame_stride,
                                          None if diag is None else diag.data_ptr(), s),
          "sobel5_launch_batch")


def launch_band(d_top, d_in, d_bot, in_pitch: int, width: int, band_rows: int, taps: Taps,
                prefetch: int, planes: dict, pitch: int, diag=None, stream=None) -> None:
    """Row band with optional 2-row halos (pointers may be peer-mapped)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    pl = planes_struct(planes, pitch)

    def ptr(x):
        if x is None:
            return None
        return x if isinstance(x, int) else x.data_ptr()

    check(_abi.load().sobel5_launch_band(ptr(d_top), ptr(d_in), ptr(d_bot), in_pitch, width,
                                         band_rows, C.byref(taps), int(prefetch), C.byref(pl),
                                         None if diag is None else diag.data_ptr(), s),
          "sobel5_launch_band")


def synth_random_device(d_img, pitch: int, width: int, height: int, seed: int = 1,
                        mask: int = 0xFF, row_offset: int = 0, stream=None) -> None:
    """synth_random (synth.hpp:20-35) generated on the GPU."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    check(_abi.load().sobel5_synth_random_device(d_img.data_ptr(), pitch, width, height,
                                                 row_offset, seed, mask, s),
          "sobel5_synth_random_device")


# ---- detect path ------------------------------------------


class SaveMode(enum.IntEnum):
    """image_io.hpp:225-228."""
    clamp_abs = 0
    normalize = 1


@dataclass
class PaddedPlane:
    """pad_replicate's result (image_io.hpp:271-277).  ``plane`` is the
    materialised (W+2r) x (H+2r) image, as in the reference; ``source`` keeps
    the unpadded image so that run_stream / detect on a PaddedPlane of radius
    2 send only the source to the GPU and pad inside the kernel's loads."""
    plane: np.ndarray
    radius: int
    source: np.ndarray | None = None

    def inner_width(self) -> int:
        return self.plane.shape[1] - 2 * self.radius

    def inner_height(self) -> int:
        return self.plane.shape[0] - 2 * self.radius


def pad_replicate(img: np.ndarray, radius: int) -> PaddedPlane:
    """image_io.hpp:279-291 (host helper, same errors and messages)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    if img.size == 0:
        raise EmptyPlane("cannot pad an empty image")
    if radius < 0:
        raise DimMismatch("pad radius must be non-negative")
    return PaddedPlane(np.pad(img, radius, mode="edge"), radius, img)


def alloc_scratch(frames: int = 1, device="cuda", out_h: int = 0, pitch: int = 0,
                  out_frame_stride: int = 0):
    """Device scratch for normalize (sobel5_detect_scratch_bytes): per-frame
    min/max + tables, plus the g^2 plane for an out_h x pitch output."""
    import torch
    n = int(_abi.load().sobel5_detect_scratch_bytes(out_h, pitch, out_frame_stride, frames))
    return torch.empty(n, dtype=torch.uint8, device=device)


def launch_ex(d_in, in_pitch: int, width: int, height: int, taps: Taps, prefetch: int,
              pad: bool, planes: dict, pitch: int, frames: int = 1, in_frame_stride: int = 0,
              out_frame_stride: int = 0, diag=None, stream=None) -> None:
    """sobel5_launch_ex: valid mode, or pad_replicate(img, 2) fused (same size)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    pl = planes_struct(planes, pitch)
    check(_abi.load().sobel5_launch_ex(d_in.data_ptr(), in_pitch, in_frame_stride, width, height,
                                       frames, C.byref(taps), int(prefetch), int(bool(pad)),
                                       C.byref(pl), out_frame_stride,
                                       None if diag is None else diag.data_ptr(), s),
          "sobel5_launch_ex")


def detect_device(d_in, in_pitch: int, width: int, height: int, taps: Taps, prefetch: int,
                  pad: bool, save_mode: SaveMode, planes: dict, pitch: int, scratch=None,
                  frames: int = 1, in_frame_stride: int = 0, out_frame_stride: int = 0,
                  diag=None, stream=None) -> None:
    """sobel5_detect: planes["u8"] = quantize(g, save_mode) of the (padded) image."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    pl = planes_struct(planes, pitch)
    check(_abi.load().sobel5_detect(d_in.data_ptr(), in_pitch, in_frame_stride, width, height,
                                    frames, C.byref(taps), int(prefetch), int(bool(pad)),
                                    int(save_mode), C.byref(pl), out_frame_stride,
                                    None if scratch is None else scratch.data_ptr(),
                                    None if diag is None else diag.data_ptr(), s),
          "sobel5_detect")


def quantize_device(d_plane, pitch: int, width: int, height: int, save_mode: SaveMode, d_u8,
                    u8_pitch: int, scratch=None, stream=None) -> None:
    """sobel5_quantize_plane on a float64 (RealPlane), int32 (SignedPlane) or
    uint8 (GrayPlane) tensor."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    kinds = {torch.float64: 0, torch.int32: 1, torch.uint8: 2}
    if d_plane.dtype not in kinds:
        raise DimMismatch("quantize needs a float64, int32 or uint8 plane")
    kind = kinds[d_plane.dtype]
    check(_abi.load().sobel5_quantize_plane(d_plane.data_ptr(), kind, pitch, width, height,
                                            int(save_mode), d_u8.data_ptr(), u8_pitch,
                                            None if scratch is None else scratch.data_ptr(), s),
          "sobel5_quantize_plane")


def quantize(plane: np.ndarray, mode: SaveMode) -> np.ndarray:
    """detail::quantize (image_io.hpp:233-256) of a host plane, computed on the GPU."""
    plane = np.ascontiguousarray(plane)
    if plane.size == 0:
        raise EmptyPlane("cannot save an empty plane")
    kinds = {np.dtype(np.float64): 0, np.dtype(np.int32): 1, np.dtype(np.uint8): 2}
    if plane.dtype not in kinds:
        raise DimMismatch("quantize needs a float64, int32 or uint8 plane")
    h, w = plane.shape
    out = np.empty((h, w), np.uint8)
    ctx = default_context()
    kind = kinds[plane.dtype]
    check(_abi.load().sobel5_quantize_host(ctx.handle, plane.ctypes.data, kind, w, h, int(mode),
                                           out.ctypes.data), f"quantize ({ctx.last_error()})")
    return out


def detect(img, params_or_taps=None, pad: bool = True, save_mode: SaveMode = SaveMode.normalize,
           prefetch: Prefetch = Prefetch.on, planes=(), ctx: Context | None = None):
    """The CLI's detect command on the GPU (sobel5_cli.cpp:127-189): optional
    pad_replicate(img, 2), run_stream, save_plane(g, save_mode).  Returns the
    u8 edge map, plus a dict of the requested planes when ``planes`` is set."""
    if isinstance(img, PaddedPlane):
        if img.radius != 2 or img.source is None:
            raise DimMismatch("detect pads by radius 2")
        img, pad = img.source, True
    taps = params_or_taps if isinstance(params_or_taps, Taps) else make_stream_taps(
        params_or_taps or FilterParams())
    ctx = ctx or default_context()
    st, u8, res, d = ctx.detect_host(np.asarray(img, dtype=np.uint8), taps, prefetch, pad,
                                     save_mode, planes)
    if st == _abi.PARITY_VIOLATION:
        raise ParityViolation(f"odd sum/difference pair ({d.sum}, {d.diff})")
    if st == _abi.EMPTY_PLANE:
        raise EmptyPlane("cannot pad an empty image")
    if st == _abi.IMAGE_TOO_SMALL:
        h, w = np.shape(img) if np.ndim(img) == 2 else (0, 0)
        raise ImageTooSmall(f"streaming filter needs at least 5x5, got {w}x{h}")
    check(st, f"detect ({ctx.last_error()})")
    return (u8, res) if planes else u8


# ---- the 3x3 operator ------------------------------------------


@dataclass
class Stream3Result:
    """pipeline.hpp:479-484."""
    gx: np.ndarray
    gy: np.ndarray
    g: np.ndarray
    counters: dict


def plan_counters_3x3(height: int, plan: StripPlan, prefetch: Prefetch) -> dict:
    widths = np.array([s.out_w for s in plan.strips], dtype=np.int32)
    c = Counters()
    check(_abi.load().sobel3_plan_counters(height, widths.ctypes.data_as(C.c_void_p),
                                           len(widths), int(prefetch), C.byref(c)),
          "plan_counters_3x3")
    return {n: int(getattr(c, n)) for n, _ in Counters._fields_}


def run_stream_3x3(img: np.ndarray, plan: StripPlan | None = None,
                   prefetch: Prefetch = Prefetch.on, workers: int = 1,
                   ctx: Context | None = None) -> Stream3Result:
    """Drop-in for sobel5::run_stream_3x3 (pipeline.hpp:551-573); ``plan``
    defaults to one full-width strip like the reference's second overload
    (:571-573)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    if img.ndim != 2:
        raise DimMismatch("image must be 2-D")
    h, w = img.shape
    if w < 3 or h < 3:  # pipeline.hpp:553-556
        raise ImageTooSmall(f"streaming filter needs at least 3x3, got {w}x{h}")
    if plan is None:
        plan = plan_strips(w, w, 1)
    if plan.in_width != w or plan.radius != 1:  # pipeline.hpp:557-560
        raise DimMismatch(f"strip plan covers {plan.in_width} columns at radius {plan.radius}, "
                          f"image has {w}")
    ctx = ctx or default_context()
    ow, oh = w - 2, h - 2
    res = {"gx": np.empty((oh, ow), np.int32), "gy": np.empty((oh, ow), np.int32),
           "g": np.empty((oh, ow), np.float64)}
    pl = Planes(pitch=ow)
    for k, v in res.items():
        setattr(pl, k, v.ctypes.data)
    st = _abi.load().sobel3_run_host(ctx.handle, img.ctypes.data, w, h, int(prefetch),
                                     C.byref(pl))
    check(st, f"run_stream_3x3 ({ctx.last_error()})")
    return Stream3Result(res["gx"], res["gy"], res["g"], plan_counters_3x3(h, plan, prefetch))


def sobel3_2d(img: np.ndarray) -> Stream3Result:
    """oracle.hpp:58-70 (identical results; computed by the streaming GPU path)."""
    return run_stream_3x3(img)


def launch3(d_in, in_pitch: int, width: int, height: int, prefetch: int, pad: bool,
            planes: dict, pitch: int, frames: int = 1, in_frame_stride: int = 0,
            out_frame_stride: int = 0, stream=None) -> None:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    pl = planes_struct(planes, pitch)
    check(_abi.load().sobel3_launch(d_in.data_ptr(), in_pitch, in_frame_stride, width, height,
                                    frames, int(prefetch), int(bool(pad)), C.byref(pl),
                                    out_frame_stride, s), "sobel3_launch")


def detect3_device(d_in, in_pitch: int, width: int, height: int, prefetch: int, pad: bool,
                   save_mode: SaveMode, planes: dict, pitch: int, scratch=None, frames: int = 1,
                   in_frame_stride: int = 0, out_frame_stride: int = 0, stream=None) -> None:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    pl = planes_struct(planes, pitch)
    check(_abi.load().sobel3_detect(d_in.data_ptr(), in_pitch, in_frame_stride, width, height,
                                    frames, int(prefetch), int(bool(pad)), int(save_mode),
                                    C.byref(pl), out_frame_stride,
                                    None if scratch is None else scratch.data_ptr(), s),
          "sobel3_detect")


# ---- one image over several GPUs from one process (config C5) -------------------

TRANSPORTS = {"auto": _abi.MGPU_AUTO, "peer": _abi.MGPU_PEER, "copy": _abi.MGPU_COPY}


class MultiGpuBands:
    """sobel5_mgpu: band k of len(devices) owns input rows [k*H/n, (k+1)*H/n)
    on devices[k] (devices may repeat); halos by peer reads inside the
    kernel or device-to-device copies."""

    def __init__(self, devices, width: int, height: int, transport: str = "auto"):
        self._lib = _abi.load()
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        check(self._lib.sobel5_mgpu_create(C.byref(h), devs, len(devices), width, height,
                                           TRANSPORTS[transport]), "sobel5_mgpu_create")
        self._h = h
        self.width, self.height, self.n = width, height, len(devices)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.sobel5_mgpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def band(self, k: int) -> dict:
        b = _abi.BandInfo()
        check(self._lib.sobel5_mgpu_band(self._h, k, C.byref(b)), "sobel5_mgpu_band")
        return {n: getattr(b, n) for n, _ in _abi.BandInfo._fields_}

    def upload(self, img: np.ndarray) -> None:
        img = np.ascontiguousarray(img, np.uint8)
        check(self._lib.sobel5_mgpu_upload(self._h, img.ctypes.data), "sobel5_mgpu_upload")

    def synth(self, seed: int, mask: int = 0xFF) -> None:
        check(self._lib.sobel5_mgpu_synth(self._h, seed, mask), "sobel5_mgpu_synth")

    def run_bands(self, taps: Taps, prefetch: int, planes: list, pitch: int) -> None:
        """planes[k]: dict of band k's device tensors (on its device)."""
        arr = (Planes * self.n)(*[planes_struct(p, pitch) for p in planes])
        check(self._lib.sobel5_mgpu_run_bands(self._h, C.byref(taps), int(prefetch), arr),
              "sobel5_mgpu_run_bands")

    def sync(self) -> None:
        check(self._lib.sobel5_mgpu_sync(self._h), "sobel5_mgpu_sync")

    def run_host(self, img: np.ndarray, taps: Taps, prefetch: Prefetch,
                 planes=("gx", "gy", "gd", "gdt", "g")) -> dict:
        img = np.ascontiguousarray(img, np.uint8)
        ow, oh = self.width - 4, self.height - 4
        dt = {"gx": np.int32, "gy": np.int32, "gd": np.int32, "gdt": np.int32, "g": np.float64,
              "g32": np.float32, "u8": np.uint8}
        res = {k: np.empty((oh, ow), dt[k]) for k in planes}
        pl = Planes(pitch=ow)
        for k, v in res.items():
            setattr(pl, k, v.ctypes.data)
        st = self._lib.sobel5_mgpu_run_host(self._h, img.ctypes.data, C.byref(taps), int(prefetch),
                                            C.byref(pl))
        if st == _abi.PARITY_VIOLATION:
            d = Diag()
            self._lib.sobel5_mgpu_last_diag(self._h, C.byref(d))
            raise ParityViolation(f"odd sum/difference pair ({d.sum}, {d.diff})")
        check(st, "sobel5_mgpu_run_host")
        return res


def run_stream_bands(img: np.ndarray, taps_or_params, plan: StripPlan, prefetch: Prefetch,
                     devices, transport: str = "auto") -> StreamResult:
    """run_stream (pipeline.hpp:452-477) with the image row-band partitioned
    over ``devices`` from this process (the C++ sobel5::run_stream_bands)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    if img.ndim != 2:
        raise DimMismatch("image must be 2-D")
    h, w = img.shape
    if w < 5 or h < 5:
        raise ImageTooSmall(f"streaming filter needs at least 5x5, got {w}x{h}")
    if plan.in_width != w or plan.radius != 2:
        raise DimMismatch(f"strip plan covers {plan.in_width} columns at radius {plan.radius}, "
                          f"image has {w}")
    taps = taps_or_params if isinstance(taps_or_params, Taps) else make_stream_taps(
        taps_or_params)
    mg = MultiGpuBands(devices, w, h, transport)
    try:
        # the plan orders the reported ParityViolation pair (strip-major)
        check(_abi.load().sobel5_mgpu_set_strip_width(mg._h, plan.lane_width - 2 * plan.radius),
              "sobel5_mgpu_set_strip_width")
        res = mg.run_host(img, taps, prefetch)
    finally:
        mg.close()
    return StreamResult(res["gx"], res["gy"], res["gd"], res["gdt"], res["g"],
                        plan_counters(h, plan, taps, prefetch))


def last_launch() -> dict:
    """Geometry of this thread's last 5x5 stencil launch (sobel5_last_launch):
    band, tma_load, kernel (index into KERNELS), grid_x/y/z."""
    info = _abi.LaunchInfo()
    check(_abi.load().sobel5_last_launch(C.byref(info)), "sobel5_last_launch")
    return {n: int(getattr(info, n)) for n, _ in _abi.LaunchInfo._fields_}


def launch_count() -> int:
    return int(_abi.load().sobel5_launch_count())
