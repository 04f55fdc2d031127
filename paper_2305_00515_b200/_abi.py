"""ctypes binding of include/sobel5_gpu.h (the product's C ABI).

Loading fails loudly if the in-tree extension is missing: there is no CPU
fallback anywhere on the product path.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

TAP_FIELDS = ("f", "h", "k0", "k1", "gx_v", "gy_v", "gdm_f", "gdm_d")


class Taps(C.Structure):
    """sobel5_taps == POD sobel5::StreamTaps (pipeline.hpp:57-73)."""

    _fields_ = [("a", C.c_int32)] + [(n, C.c_int32 * 5) for n in TAP_FIELDS] + [
        ("wide_vagg", C.c_int32)]

    def as_dict(self) -> dict:
        d = {"a": int(self.a), "wide_vagg": int(self.wide_vagg)}
        for n in TAP_FIELDS:
            d[n] = [int(v) for v in getattr(self, n)]
        return d

    @classmethod
    def from_dict(cls, d: dict) -> "Taps":
        t = cls()
        t.a = int(d["a"])
        t.wide_vagg = int(d.get("wide_vagg", 0))
        for n in TAP_FIELDS:
            getattr(t, n)[:] = [int(v) for v in d[n]]
        return t

    def copy(self) -> "Taps":
        return Taps.from_dict(self.as_dict())

    def __eq__(self, other):
        return isinstance(other, Taps) and self.as_dict() == other.as_dict()


class Planes(C.Structure):
    _fields_ = [("gx", C.c_void_p), ("gy", C.c_void_p), ("gd", C.c_void_p), ("gdt", C.c_void_p),
                ("g", C.c_void_p), ("g32", C.c_void_p), ("u8", C.c_void_p),
                ("pitch", C.c_int64)]


class Diag(C.Structure):
    _fields_ = [("violations", C.c_int32), ("strip_w", C.c_int32), ("reserved", C.c_int32 * 2),
                ("order", C.c_uint64), ("sum", C.c_int32), ("diff", C.c_int32)]


# int32 words of a device-side sobel5_diag (a torch.int32 tensor of this many
# elements; word 0 = violations, 1 = strip_w, 6 = sum, 7 = diff)
DIAG_WORDS = 8


class IpcHandle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 64), ("offset", C.c_int64)]


class LaunchInfo(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("band", "tma_load", "kernel", "grid_x", "grid_y",
                                         "grid_z")]


class BandInfo(C.Structure):
    _fields_ = [("device", C.c_int), ("r0", C.c_int), ("r1", C.c_int), ("out_row0", C.c_int),
                ("out_rows", C.c_int), ("d_in", C.c_void_p), ("in_pitch", C.c_int64),
                ("stream", C.c_void_p), ("transport", C.c_int)]


class Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "row_conv5_f", "row_conv5_h", "row_conv5_k0", "row_conv5_k1",
        "row_diff", "row_conv3_f", "row_conv3_h", "mac")]


MGPU_AUTO, MGPU_PEER, MGPU_COPY = -1, 0, 1

PLANE_NAMES = ("gx", "gy", "gd", "gdt", "g", "g32", "u8")

# sobel5_status
OK, IMAGE_TOO_SMALL, DIM_MISMATCH, PARITY_VIOLATION, INVALID_ARG, CUDA_ERROR, \
    OUT_OF_MEMORY, NON_POSITIVE_PARAM, PARAM_OVERFLOW, LANE_TOO_NARROW, NO_DEVICE, \
    EMPTY_PLANE = range(12)

EXPORTS = (
    "sobel5_abi_version", "sobel5_status_string", "sobel5_launch_count", "sobel5_make_taps",
    "sobel5_plan_counters", "sobel5_launch", "sobel5_launch_batch", "sobel5_launch_band",
    "sobel5_synth_random_device", "sobel5_ctx_create", "sobel5_ctx_destroy",
    "sobel5_ctx_last_error", "sobel5_run_host", "sobel5_selftest", "sobel5_ipc_export",
    "sobel5_ipc_import", "sobel5_ipc_release", "sobel5_launch_ex", "sobel5_detect",
    "sobel5_detect_scratch_bytes", "sobel5_quantize_plane", "sobel5_detect_host",
    "sobel3_launch", "sobel3_detect", "sobel3_plan_counters", "sobel3_run_host",
    "sobel5_quantize_host", "sobel5_run_host_begin", "sobel5_run_host_finish",
    "sobel5_run_host_chunk", "sobel5_run_host_staging", "sobel5_run_host_staging_elem",
    "sobel5_kernel_for_taps",
    "sobel3_run_host_begin", "sobel5_ctx_trim", "sobel5_last_launch",
    "sobel5_ctx_set_strip_width", "sobel5_ctx_last_d2h_bytes", "sobel5_run_host_frames",
    "sobel5_conv2d_valid", "sobel5_conv2d_valid_host", "sobel5_dense_4d", "sobel5_dense_4d_host",
    "sobel5_mgpu_create", "sobel5_mgpu_destroy", "sobel5_mgpu_band", "sobel5_mgpu_upload",
    "sobel5_mgpu_synth", "sobel5_mgpu_run_bands", "sobel5_mgpu_sync", "sobel5_mgpu_run_host", "sobel5_mgpu_last_diag",
    "sobel5_mgpu_set_strip_width",
    "sobel5_host_register", "sobel5_host_unregister", "sobel5_stream_write_u32",
    "sobel5_stream_wait_u32",
)

_lib = None


def lib_path() -> str:
    # SOBEL5_LIB: an alternative in-tree build (tools/build_variant.sh, A/B experiments)
    return os.environ.get("SOBEL5_LIB") or _build.LIB


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load libsobel5_b200.so (building it in-tree first if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        if not build_if_missing:
            raise RuntimeError(f"sobel5 CUDA extension missing: {path}")
        _build.build()
    L = C.CDLL(path)
    vp, i32, i64 = C.c_void_p, C.c_int, C.c_int64
    L.sobel5_abi_version.restype = i32
    L.sobel5_status_string.argtypes = [i32]
    L.sobel5_status_string.restype = C.c_char_p
    L.sobel5_launch_count.restype = C.c_uint64
    L.sobel5_last_launch.argtypes = [C.POINTER(LaunchInfo)]
    L.sobel5_last_launch.restype = i32
    L.sobel5_conv2d_valid.argtypes = [vp, i64, i32, i32, vp, i32, vp, i64, vp]
    L.sobel5_conv2d_valid.restype = i32
    L.sobel5_conv2d_valid_host.argtypes = [vp, vp, i32, i32, vp, i32, vp]
    L.sobel5_conv2d_valid_host.restype = i32
    L.sobel5_dense_4d.argtypes = [vp, i64, i32, i32, vp, C.POINTER(Planes), vp]
    L.sobel5_dense_4d.restype = i32
    L.sobel5_dense_4d_host.argtypes = [vp, vp, i32, i32, vp, C.POINTER(Planes)]
    L.sobel5_dense_4d_host.restype = i32
    L.sobel5_mgpu_create.argtypes = [C.POINTER(vp), vp, i32, i32, i32, i32]
    L.sobel5_mgpu_create.restype = i32
    L.sobel5_mgpu_destroy.argtypes = [vp]
    L.sobel5_mgpu_destroy.restype = None
    L.sobel5_mgpu_band.argtypes = [vp, i32, C.POINTER(BandInfo)]
    L.sobel5_mgpu_band.restype = i32
    L.sobel5_mgpu_upload.argtypes = [vp, vp]
    L.sobel5_mgpu_upload.restype = i32
    L.sobel5_mgpu_synth.argtypes = [vp, C.c_uint64, C.c_uint8]
    L.sobel5_mgpu_synth.restype = i32
    L.sobel5_mgpu_run_bands.argtypes = [vp, C.POINTER(Taps), i32, vp]
    L.sobel5_mgpu_run_bands.restype = i32
    L.sobel5_mgpu_sync.argtypes = [vp]
    L.sobel5_mgpu_sync.restype = i32
    L.sobel5_mgpu_run_host.argtypes = [vp, vp, C.POINTER(Taps), i32, C.POINTER(Planes)]
    L.sobel5_mgpu_run_host.restype = i32
    L.sobel5_mgpu_last_diag.argtypes = [vp, C.POINTER(Diag)]
    L.sobel5_mgpu_last_diag.restype = i32
    L.sobel5_mgpu_set_strip_width.argtypes = [vp, i32]
    L.sobel5_mgpu_set_strip_width.restype = i32
    L.sobel5_host_register.argtypes = [vp, C.c_size_t, C.POINTER(vp)]
    L.sobel5_host_register.restype = i32
    L.sobel5_host_unregister.argtypes = [vp]
    L.sobel5_host_unregister.restype = i32
    L.sobel5_stream_write_u32.argtypes = [vp, C.c_uint32, vp]
    L.sobel5_stream_write_u32.restype = i32
    L.sobel5_stream_wait_u32.argtypes = [vp, C.c_uint32, vp]
    L.sobel5_stream_wait_u32.restype = i32
    L.sobel5_make_taps.argtypes = [i64] * 4 + [C.POINTER(Taps)]
    L.sobel5_make_taps.restype = i32
    L.sobel5_plan_counters.argtypes = [i32, vp, i32, C.POINTER(Taps), i32, C.POINTER(Counters)]
    L.sobel5_plan_counters.restype = i32
    L.sobel5_launch.argtypes = [vp, i64, i32, i32, C.POINTER(Taps), i32, C.POINTER(Planes), vp,
                                vp]
    L.sobel5_launch.restype = i32
    L.sobel5_launch_batch.argtypes = [vp, i64, i64, i32, i32, i32, C.POINTER(Taps), i32,
                                      C.POINTER(Planes), i64, vp, vp]
    L.sobel5_launch_batch.restype = i32
    L.sobel5_launch_band.argtypes = [vp, vp, vp, i64, i32, i32, C.POINTER(Taps), i32,
                                     C.POINTER(Planes), vp, vp]
    L.sobel5_launch_band.restype = i32
    L.sobel5_synth_random_device.argtypes = [vp, i64, i32, i32, i64, C.c_uint64, C.c_uint8, vp]
    L.sobel5_synth_random_device.restype = i32
    L.sobel5_ctx_create.argtypes = [C.POINTER(vp), i32]
    L.sobel5_ctx_create.restype = i32
    L.sobel5_ctx_destroy.argtypes = [vp]
    L.sobel5_ctx_destroy.restype = None
    L.sobel5_ctx_last_error.argtypes = [vp]
    L.sobel5_ctx_last_error.restype = C.c_char_p
    L.sobel5_run_host.argtypes = [vp, vp, i32, i32, C.POINTER(Taps), i32, C.POINTER(Planes),
                                  C.POINTER(Diag)]
    L.sobel5_run_host.restype = i32
    L.sobel5_run_host_begin.argtypes = [vp, vp, i32, i32, C.POINTER(Taps), i32, C.c_uint32]
    L.sobel5_run_host_begin.restype = i32
    L.sobel5_run_host_finish.argtypes = [vp, C.POINTER(Planes), C.POINTER(Diag)]
    L.sobel5_run_host_finish.restype = i32
    L.sobel5_ctx_trim.argtypes = [vp]
    L.sobel5_ctx_trim.restype = None
    L.sobel5_ctx_set_strip_width.argtypes = [vp, i32]
    L.sobel5_ctx_set_strip_width.restype = i32
    L.sobel5_ctx_last_d2h_bytes.argtypes = [vp]
    L.sobel5_ctx_last_d2h_bytes.restype = C.c_uint64
    L.sobel5_run_host_frames.argtypes = [vp, vp, i32, i32, i32, C.c_int64, C.POINTER(Taps), i32,
                                         C.POINTER(Planes), C.c_int64, vp]
    L.sobel5_run_host_frames.restype = i32
    L.sobel3_run_host_begin.argtypes = [vp, vp, i32, i32, i32, C.c_uint32]
    L.sobel3_run_host_begin.restype = i32
    L.sobel5_kernel_for_taps.argtypes = [C.POINTER(Taps)]
    L.sobel5_kernel_for_taps.restype = i32
    L.sobel5_run_host_chunk.argtypes = [vp, i32, C.POINTER(i32), C.POINTER(i32)]
    L.sobel5_run_host_chunk.restype = i32
    L.sobel5_run_host_staging.argtypes = [vp, i32]
    L.sobel5_run_host_staging.restype = vp
    L.sobel5_run_host_staging_elem.argtypes = [vp, i32]
    L.sobel5_run_host_staging_elem.restype = i32
    L.sobel5_ipc_export.argtypes = [vp, C.POINTER(IpcHandle)]
    L.sobel5_ipc_export.restype = i32
    L.sobel5_ipc_import.argtypes = [C.POINTER(IpcHandle), C.POINTER(vp)]
    L.sobel5_ipc_import.restype = i32
    L.sobel5_ipc_release.argtypes = [vp]
    L.sobel5_ipc_release.restype = i32
    L.sobel5_selftest.argtypes = [i32, C.c_uint32, C.c_uint32, vp, vp]
    L.sobel5_selftest.restype = i32
    L.sobel5_launch_ex.argtypes = [vp, i64, i64, i32, i32, i32, C.POINTER(Taps), i32, i32,
                                   C.POINTER(Planes), i64, vp, vp]
    L.sobel5_launch_ex.restype = i32
    L.sobel5_detect_scratch_bytes.argtypes = [i32, i64, i64, i32]
    L.sobel5_detect_scratch_bytes.restype = C.c_size_t
    L.sobel5_detect.argtypes = [vp, i64, i64, i32, i32, i32, C.POINTER(Taps), i32, i32, i32,
                                C.POINTER(Planes), i64, vp, vp, vp]
    L.sobel5_detect.restype = i32
    L.sobel5_quantize_plane.argtypes = [vp, i32, i64, i32, i32, i32, vp, i64, vp, vp]
    L.sobel5_quantize_plane.restype = i32
    L.sobel5_detect_host.argtypes = [vp, vp, i32, i32, C.POINTER(Taps), i32, i32, i32, vp,
                                     C.POINTER(Planes), C.POINTER(Diag)]
    L.sobel5_detect_host.restype = i32
    L.sobel3_launch.argtypes = [vp, i64, i64, i32, i32, i32, i32, i32, C.POINTER(Planes), i64,
                                vp]
    L.sobel3_launch.restype = i32
    L.sobel3_detect.argtypes = [vp, i64, i64, i32, i32, i32, i32, i32, i32, C.POINTER(Planes),
                                i64, vp, vp]
    L.sobel3_detect.restype = i32
    L.sobel3_plan_counters.argtypes = [i32, vp, i32, i32, C.POINTER(Counters)]
    L.sobel3_plan_counters.restype = i32
    L.sobel3_run_host.argtypes = [vp, vp, i32, i32, i32, C.POINTER(Planes)]
    L.sobel3_run_host.restype = i32
    L.sobel5_quantize_host.argtypes = [vp, vp, i32, i32, i32, i32, vp]
    L.sobel5_quantize_host.restype = i32
    _lib = L
    return L


def status_string(code: int) -> str:
    return load().sobel5_status_string(code).decode()
