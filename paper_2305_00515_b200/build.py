"""In-tree build of the sm_100a extension (no JIT cache, no pip install).

``python -m paper_2305_00515_b200.build`` compiles csrc/*.cu with nvcc into
paper_2305_00515_b200/lib/libsobel5_b200.so.  The .so is git-ignored but
travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libsobel5_b200.so")
SOURCES = ["sobel5_abi.cu", "sobel5_ctx.cu", "sobel5_ipc.cu", "sobel5_detect.cu",
           "sobel5_k_plain.cu", "sobel5_k_seg.cu", "sobel5_k_pad.cu", "sobel5_k_generic.cu",
           "sobel3_k.cu", "sobel5_k_rtaps.cu", "sobel5_k_f32.cu", "sobel5_k_dense.cu",
           "sobel5_conv2d.cu", "sobel5_mgpu.cu", "sobel5_k_u8.cu", "sobel5_tmap.cu",
           "sobel3_k_u8.cu", "sobel5_wire.cpp"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
# host-only translation units (.cpp) go through nvcc to the host compiler

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                     "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
OBJDIR = os.path.join(ROOT, "build", "obj")


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "sobel5_gpu.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Each translation unit compiles in its own nvcc process (in parallel),
    then one nvcc link produces the shared library."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    nv = nvcc()

    def compile_one(src):
        obj = os.path.join(OBJDIR, os.path.splitext(src)[0] + ".o")
        extra = os.environ.get("SOBEL5_NVCC_EXTRA", "").split()
        cmd = [nv] + NVCC_FLAGS + extra + (["-Xptxas=-v"] if verbose else []) + [
            "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {src}")
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + ".tmp"
    subprocess.run([nv] + ARCH + ["-shared", "-o", tmp] + objs, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
