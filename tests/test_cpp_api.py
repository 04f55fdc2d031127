"""The drop-in C++ API (include/sobel5_b200/*.hpp) through its own test
program tests/cpp/test_api.cpp: host-side checks on CPU, run_stream on GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "test_api")


@pytest.fixture(scope="module")
def exe():
    from paper_2305_00515_b200 import _abi
    _abi.load()  # builds the .so in-tree if missing
    srcs = [os.path.join(ROOT, "tests", "cpp", "test_api.cpp")] + [
        os.path.join(ROOT, "include", "sobel5_b200", f)
        for f in os.listdir(os.path.join(ROOT, "include", "sobel5_b200"))]
    if not os.path.exists(EXE) or any(os.path.getmtime(s) > os.path.getmtime(EXE) for s in srcs):
        subprocess.run(["bash", os.path.join(ROOT, "tools", "build_cpp.sh")], check=True)
    return EXE


def test_cpp_api_host(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_api_gpu(exe, cuda):
    r = subprocess.run([exe, "--gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_api_gpu_staging_cap(exe, cuda):
    """The same checks with a 1 MB pinned-staging cap: larger results take
    the direct-download fallback of run_stream / run_stream_3x3."""
    env = dict(os.environ, SOBEL5_STAGING_MAX_MB="1")
    r = subprocess.run([exe, "--gpu"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("wire", ["1", "0"])
def test_cpp_api_gpu_wire(exe, cuda, wire):
    """The same checks with the int16 wire on (the default: the C++
    run_stream sign-extends gx..gdt from the int16 staging) and off."""
    env = dict(os.environ, SOBEL5_WIRE16=wire)
    r = subprocess.run([exe, "--gpu"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
