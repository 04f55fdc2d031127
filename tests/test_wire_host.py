"""CPU: the host side of the int16 D2H wire (sobel5_wire.cpp) -- widening and
the magnitude plane rebuilt from the int16 gradients -- equal to the
reference's formula bit for bit (tests/cpp/wire_decode_check.cpp, built here
with g++ from the library's own source; no GPU)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
@pytest.mark.parametrize("isa", ["", "avx2", "scalar"])
def test_wire_decode(tmp_path, isa):
    exe = str(tmp_path / "wire_decode_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-o", exe,
                    os.path.join(ROOT, "tests", "cpp", "wire_decode_check.cpp"),
                    os.path.join(ROOT, "paper_2305_00515_b200", "csrc", "sobel5_wire.cpp")],
                   check=True)
    env = dict(os.environ, SOBEL5_WIRE_ISA=isa)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
