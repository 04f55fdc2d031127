"""Generates tests/golden/png/: PNG and PGM files plus manifest.json, the
expected result of the reference's load_gray on each (image_io.hpp:20-213).

The reference decodes PNG with libpng, which is not available to C++ here;
the expected planes come from libpng itself through OpenCV (cv2.imread,
IMREAD_UNCHANGED: libpng's decode, channels reordered from BGR(A)) reduced
with the reference's integer BT.601 luma, (77 R + 150 G + 29 B + 128) >> 8.
Files libpng cannot write here (Adam7 interlace, chosen filters, split IDAT,
ancillary chunks, palette, gray+alpha, deliberate corruption) come from the
small encoder below, and every one of them that libpng can read is checked
to decode through libpng to the pixels it was made from.  Error cases carry
the exception type and message the reference raises ({path} = the path
passed to load_gray).  Run: python tests/golden/make_png_fixtures.py"""
import json
import os
import struct
import zlib

import cv2
import numpy as np

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "png")
ADAM7 = [(0, 0, 8, 8), (4, 0, 8, 8), (0, 4, 4, 8), (2, 0, 4, 4), (0, 2, 2, 4), (1, 0, 2, 2), (0, 1, 1, 2)]


def fnv(b):
    h = 1469598103934665603
    for x in bytes(b):
        h = ((h ^ x) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def chunk(t, d):
    return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xFFFFFFFF)


def paeth(a, b, c):
    p = a + b - c
    pa, pb, pc = abs(p - a), abs(p - b), abs(p - c)
    return a if pa <= pb and pa <= pc else (b if pb <= pc else c)


def filt(rows, bpp, ftype):
    """Scanlines of one pass with filter ftype(y) per row."""
    out, prev = bytearray(), None
    for y, row in enumerate(rows):
        f = ftype(y)
        r = bytearray(len(row))
        for i, v in enumerate(row):
            a = row[i - bpp] if i >= bpp else 0
            b = prev[i] if prev is not None else 0
            c = prev[i - bpp] if prev is not None and i >= bpp else 0
            pred = [0, a, b, (a + b) >> 1, paeth(a, b, c)][f] if f < 5 else 0
            r[i] = (v - pred) & 0xFF
        out += bytes([f]) + r
        prev = row
    return bytes(out)


def encode(px, ct, depth=8, interlace=False, ftype=lambda y: y % 5, idat_split=None, extra=(),
           plte=None):
    """px: (h, w, ch) uint8 (ch = 1/2/3/4) -> PNG bytes."""
    h, w = px.shape[:2]
    ch = px.shape[2]
    raw = b""
    passes = ADAM7 if interlace else [(0, 0, 1, 1)]
    for x0, y0, dx, dy in passes:
        sub = px[y0::dy, x0::dx]
        if sub.shape[0] == 0 or sub.shape[1] == 0:
            continue
        raw += filt([bytes(r.reshape(-1)) for r in sub], ch, ftype)
    z = zlib.compress(raw, 9)
    ihdr = struct.pack(">IIBBBBB", w, h, depth, ct, 0, 0, 1 if interlace else 0)
    body = chunk(b"IHDR", ihdr)
    for t, d in extra:
        body += chunk(t, d)
    if plte is not None:
        body += chunk(b"PLTE", plte)
    parts = [z] if not idat_split else [z[i:i + idat_split] for i in range(0, len(z), idat_split)]
    for p in parts:
        body += chunk(b"IDAT", p)
    return b"\x89PNG\r\n\x1a\n" + body + chunk(b"IEND", b"")


def libpng_gray(path):
    """libpng's decode (cv2) reduced like the reference's load_png."""
    a = cv2.imread(path, cv2.IMREAD_UNCHANGED)
    assert a is not None and a.dtype == np.uint8, path
    if a.ndim == 2:
        return a
    b, g, r = (a[..., i].astype(np.int32) for i in range(3))
    return ((77 * r + 150 * g + 29 * b + 128) >> 8).astype(np.uint8)


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(2305)
    man = {}

    def ok(name, data=None, writer=None, src=None):
        path = os.path.join(OUT, name)
        if writer:
            writer(path)
        else:
            open(path, "wb").write(data)
        g = libpng_gray(path) if name.endswith(".png") else src
        if src is not None and name.endswith(".png"):
            # the file decodes through libpng to the pixels it was made from
            s = src if src.ndim == 2 else None
            if s is not None:
                assert np.array_equal(g, s), name
        man[name] = {"w": int(g.shape[1]), "h": int(g.shape[0]), "fnv": fnv(g.tobytes())}

    def err(name, data, kind, msg):
        open(os.path.join(OUT, name), "wb").write(data)
        man[name] = {"error": f"{kind}: {msg}"}

    # libpng-written (cv2) 8-bit gray / RGB / RGBA, no interlace
    g = rng.integers(0, 256, (23, 37), dtype=np.uint8)
    ok("cv_gray.png", writer=lambda p: cv2.imwrite(p, g), src=g)
    rgb = rng.integers(0, 256, (17, 41, 3), dtype=np.uint8)
    ok("cv_rgb.png", writer=lambda p: cv2.imwrite(p, rgb))
    rgba = rng.integers(0, 256, (31, 29, 4), dtype=np.uint8)
    ok("cv_rgba.png", writer=lambda p: cv2.imwrite(p, rgba))
    smooth = (np.add.outer(np.arange(40), np.arange(60)) * 3 % 256).astype(np.uint8)
    ok("cv_smooth.png", writer=lambda p: cv2.imwrite(p, smooth, [cv2.IMWRITE_PNG_COMPRESSION, 9]), src=smooth)

    # own encoder: every filter type, Adam7, split IDAT, ancillary chunks, tiny sizes
    for name, shape, ct, il in [("f_gray.png", (19, 23, 1), 0, False), ("i_gray.png", (35, 33, 1), 0, True),
                                ("i_rgb.png", (13, 19, 3), 2, True), ("i_rgba.png", (9, 10, 4), 6, True),
                                ("f_rgb.png", (11, 7, 3), 2, False), ("t_1x1.png", (1, 1, 1), 0, True),
                                ("t_9x1.png", (1, 9, 1), 0, False), ("t_1x9.png", (9, 1, 1), 0, True),
                                ("t_3x2_rgb.png", (2, 3, 3), 2, True)]:
        px = rng.integers(0, 256, shape, dtype=np.uint8)
        data = encode(px, ct, interlace=il)
        src = px[..., 0] if shape[2] == 1 else None
        ok(name, data, src=src)
        if shape[2] == 3:  # colour: the expected plane is libpng's decode + luma
            pass
    px = rng.integers(0, 256, (40, 50, 1), dtype=np.uint8)
    ok("split_idat_text.png", encode(px, 0, idat_split=97,
                                     extra=[(b"tEXt", b"Comment\x00made for the tests"),
                                            (b"gAMA", struct.pack(">I", 45455))]), src=px[..., 0])
    # an ancillary chunk with a bad CRC is discarded (a libpng warning)
    d = bytearray(encode(px, 0, extra=[(b"tEXt", b"Title\x00x")]))
    i = d.index(b"tEXt")
    d[i + 4 + 7] ^= 0xFF  # corrupt the CRC (4 type + 7 data bytes in)
    ok("bad_crc_ancillary.png", bytes(d), src=px[..., 0])
    # trailing garbage after IEND is never read
    ok("after_iend.png", encode(px, 0) + b"garbage", src=px[..., 0])

    # the reference's rejections (image_io.hpp:105-117), in its order
    g16 = rng.integers(0, 65536, (8, 8), dtype=np.uint16)
    p16 = os.path.join(OUT, "depth16.png")
    cv2.imwrite(p16, g16)
    man["depth16.png"] = {"error": "UnsupportedFormat: PNG bit depth 16 in {path}, only 8 is supported"}
    pal = rng.integers(0, 4, (6, 6, 1), dtype=np.uint8)
    err("palette.png", encode(pal, 3, plte=bytes(range(12))), "UnsupportedFormat",
        "PNG color type 3 in {path}, need gray, RGB or RGBA")
    err("gray_alpha.png", encode(rng.integers(0, 256, (5, 4, 2), dtype=np.uint8), 4), "UnsupportedFormat",
        "PNG color type 4 in {path}, need gray, RGB or RGBA")
    err("gray4.png", encode(rng.integers(0, 16, (4, 4, 1), dtype=np.uint8), 0, depth=4),
        "UnsupportedFormat", "PNG bit depth 4 in {path}, only 8 is supported")
    # depth / colour type are checked before the image data are read
    d16 = open(p16, "rb").read()
    err("depth16_truncated.png", d16[: len(d16) - 20], "UnsupportedFormat",
        "PNG bit depth 16 in {path}, only 8 is supported")
    # what libpng rejects while reading
    good = encode(px, 0)
    err("bad_sig.png", b"\x89PXG\r\n\x1a\n" + good[8:], "CorruptFile", "bad PNG signature in {path}")
    d = bytearray(good)
    i = d.index(b"IDAT")
    d[i + 10] ^= 0x55  # data byte, CRC now wrong
    err("bad_crc_idat.png", bytes(d), "CorruptFile", "libpng failed to decode {path}")
    err("truncated.png", good[: len(good) // 2], "CorruptFile", "libpng failed to decode {path}")
    err("no_iend.png", good[:-12], "CorruptFile", "libpng failed to decode {path}")
    err("bad_ihdr_depth.png", encode(px, 0, depth=3), "CorruptFile", "libpng failed to decode {path}")
    err("bad_filter.png", encode(px, 0, ftype=lambda y: 5 if y == 7 else 0), "CorruptFile",
        "libpng failed to decode {path}")
    short = px[:20]  # IHDR says 40 rows, the data hold 20
    hdr = struct.pack(">IIBBBBB", 50, 40, 8, 0, 0, 0, 0)
    z = zlib.compress(filt([bytes(r.reshape(-1)) for r in short], 1, lambda y: 0))
    err("short_data.png", b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", hdr) + chunk(b"IDAT", z) + chunk(b"IEND", b""),
        "CorruptFile", "libpng failed to decode {path}")
    err("bad_zlib.png", b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", hdr) + chunk(b"IDAT", b"\x78\x9c\xff\xff\xff")
        + chunk(b"IEND", b""), "CorruptFile", "libpng failed to decode {path}")
    err("unknown_critical.png", good[:33] + chunk(b"ABCD", b"xyz") + good[33:], "CorruptFile",
        "libpng failed to decode {path}")
    err("no_idat.png", b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", hdr) + chunk(b"IEND", b""), "CorruptFile",
        "libpng failed to decode {path}")

    # PGM (image_io.hpp:27-72, 216-223)
    pg = rng.integers(0, 256, (7, 11), dtype=np.uint8)
    ok("p5.pgm", b"P5\n11 7\n255\n" + pg.tobytes(), src=pg)
    ok("p5_comments.pgm", b"P5\n# made by\n# the tests\n11\t7 \n255\n" + pg.tobytes(), src=pg)
    p2 = "P2\n# ascii\n11 7\n255\n" + "\n".join(" ".join(str(v) for v in r) for r in pg) + "\n"
    ok("p2.pgm", p2.encode(), src=pg)
    err("p5_maxval.pgm", b"P5\n2 2\n65535\n" + bytes(8), "UnsupportedFormat",
        "PGM maxval 65535 in {path}, only 255 is supported")
    err("p5_dims.pgm", b"P5\n0 2\n255\n", "CorruptFile", "bad PGM dimensions in {path}")
    err("p5_short.pgm", b"P5\n4 4\n255\n" + bytes(10), "CorruptFile", "truncated PGM pixel data in {path}")
    err("p2_range.pgm", b"P2\n2 1\n255\n12 300\n", "CorruptFile", "PGM sample 300 out of range in {path}")
    err("p2_short.pgm", b"P2\n2 2\n255\n1 2 3\n", "CorruptFile", "truncated PGM pixel data in {path}")
    err("p2_header.pgm", b"P2\n# c\nabc 2\n255\n", "CorruptFile", "malformed PGM header")
    err("p5_header_eof.pgm", b"P5\n12", "CorruptFile", "truncated PGM header")
    err("gif.gif", b"GIF89a" + bytes(20), "UnsupportedFormat", "unrecognized image format in {path}")
    man["missing.png"] = {"error": "IoError: cannot open {path}"}

    json.dump(man, open(os.path.join(OUT, "manifest.json"), "w"), indent=1, sort_keys=True)
    print(len(man), "fixtures")


if __name__ == "__main__":
    main()
