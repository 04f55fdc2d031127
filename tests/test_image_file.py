"""CPU: the image files either side of the path (SURVEY 8f row 4's data
formats; image_io.hpp:20-223) through the drop-in headers
(include/sobel5_b200/image_file.hpp: PGM, and PNG on zlib instead of
libpng).  load_gray must give every fixture of tests/golden/png the plane
libpng decodes (BT.601 luma for colour) or the reference's exception type
and message; save_gray's PNG must decode through libpng (OpenCV) to the
plane, its PGM must be the reference's bytes.  No GPU."""
import json
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "png")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    out = str(tmp_path_factory.mktemp("imf") / "image_file_check")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"), "-o", out,
                    os.path.join(ROOT, "tests", "cpp", "image_file_check.cpp"),
                    "-L", os.path.join(ROOT, "paper_2305_00515_b200", "lib"), "-lsobel5_b200", "-lz",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_2305_00515_b200", "lib")], check=True)
    return out


def test_load_gray_fixtures(exe):
    man = json.load(open(os.path.join(GOLD, "manifest.json")))
    names = sorted(man)
    paths = [os.path.join(GOLD, n) for n in names]
    r = subprocess.run([exe, "load", *paths], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    got = r.stdout.splitlines()
    assert len(got) == len(names)
    for n, p, line in zip(names, paths, got):
        m = man[n]
        want = (m["error"].format(path=p) if "error" in m else f"ok {m['w']}x{m['h']} {m['fnv']}")
        assert line == want, n


def _fnv(b):
    h = 1469598103934665603
    for x in bytes(b):
        h = ((h ^ x) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


@pytest.mark.parametrize("w,h,kind", [(1, 1, "rand"), (37, 5, "rand"), (256, 97, "smooth"),
                                      (640, 480, "rand"), (33, 1, "flat")])
def test_save_gray_roundtrip(exe, tmp_path, w, h, kind):
    cv2 = pytest.importorskip("cv2")
    rng = np.random.default_rng(w * h)
    if kind == "rand":
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
    elif kind == "smooth":
        img = (np.add.outer(np.arange(h), 2 * np.arange(w)) % 256).astype(np.uint8)
    else:
        img = np.full((h, w), 77, np.uint8)
    raw = tmp_path / "in.raw"
    raw.write_bytes(img.tobytes())
    outs = [str(tmp_path / n) for n in ("o.png", "o.PNG", "o.pgm", "o.Pgm", "o.bmp")]
    r = subprocess.run([exe, "save", str(raw), str(w), str(h), *outs], capture_output=True, text=True,
                       timeout=60)
    assert r.stdout.splitlines() == ["ok"] * 4 + [
        f"UnsupportedExtension: cannot infer image format from {outs[4]}"]
    for p in outs[:2]:  # libpng reads the plane back; so does load_gray
        back = cv2.imread(p, cv2.IMREAD_UNCHANGED)
        assert back is not None and back.shape == (h, w) and np.array_equal(back, img)
    for p in outs[2:4]:  # the reference's P5 bytes (image_io.hpp:216-223)
        assert open(p, "rb").read() == f"P5\n{w} {h}\n255\n".encode() + img.tobytes()
    r = subprocess.run([exe, "load", *outs[:4]], capture_output=True, text=True, timeout=60)
    assert r.stdout.splitlines() == [f"ok {w}x{h} {_fnv(img.tobytes())}"] * 4


def test_save_gray_unwritable(exe, tmp_path):
    raw = tmp_path / "in.raw"
    raw.write_bytes(bytes(4))
    bad = str(tmp_path / "no_such_dir" / "x.png")
    bad2 = str(tmp_path / "no_such_dir" / "x.pgm")
    r = subprocess.run([exe, "save", str(raw), "2", "2", bad, bad2], capture_output=True, text=True)
    assert r.stdout.splitlines() == [f"IoError: cannot write {bad}", f"IoError: cannot write {bad2}"]


def test_load_gray_mutations(exe, tmp_path):
    """Random byte flips and truncations of valid files: every load ends in a
    plane or one of the reference's exceptions, never a crash."""
    rng = np.random.default_rng(7)
    paths = []
    for src in ("cv_rgb.png", "i_gray.png", "split_idat_text.png", "p5.pgm", "p2.pgm"):
        data = open(os.path.join(GOLD, src), "rb").read()
        for k in range(40):
            d = bytearray(data)
            if k % 4 == 3:
                d = d[: int(rng.integers(1, len(d)))]
            else:
                for _ in range(int(rng.integers(1, 4))):
                    d[int(rng.integers(0, len(d)))] = int(rng.integers(0, 256))
            p = tmp_path / f"{src}.{k}"
            p.write_bytes(bytes(d))
            paths.append(str(p))
    r = subprocess.run([exe, "load", *paths], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert len(lines) == len(paths)
    for line in lines:
        assert line.startswith(("ok ", "CorruptFile: ", "UnsupportedFormat: ")), line
