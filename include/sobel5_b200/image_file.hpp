// sobel5_b200/image_file.hpp -- the image files either side of the path:
// 8-bit grayscale PGM (P2 / P5) and PNG load / save, integer BT.601 luma.
//
// Restates the behaviour of the reference's file I/O (image_io.hpp:20-223)
// without libpng: PNG is decoded and encoded here on top of zlib (link -lz),
// with the reference's accepted formats, exception types and messages:
//   * load_gray sniffs the first two bytes: "P2" / "P5" -> PGM, 0x89 'P' ->
//     PNG, anything else UnsupportedFormat (image_io.hpp:201-213);
//   * PGM: whitespace and '#' comment lines between header values, maxval
//     255 only, P5 pixel bytes after one whitespace byte, P2 decimal samples
//     in [0, maxval] (image_io.hpp:27-72);
//   * PNG: 8-bit gray, RGB or RGBA, interlaced or not (libpng's interlace
//     handling, image_io.hpp:119), colour reduced with luma_bt601; other bit
//     depths / colour types are UnsupportedFormat in the order the reference
//     checks them (image_io.hpp:105-117); anything libpng rejects while
//     reading -- a bad IHDR, a CRC error in a critical chunk, an unknown
//     critical chunk, a zlib error, missing image data, a bad filter byte, a
//     file that ends before IEND -- is CorruptFile("libpng failed to decode
//     <path>") as the reference's setjmp handler reports it (image_io.hpp:97);
//   * save_gray picks the format by extension, case-insensitively (PGM P5 or
//     8-bit gray PNG), else UnsupportedExtension (image_io.hpp:216-223).
//     The PNG encoder filters each row with libpng's default heuristic
//     (minimum sum of absolute signed residuals over None / Sub / Up /
//     Average / Paeth) and deflates at zlib's default level; its bytes need
//     not equal libpng's, the pixels any PNG decoder reads back are the
//     plane's (tests/test_image_file.py checks both directions against
//     libpng).
#pragma once

#include <zlib.h>

#include <algorithm>
#include <array>
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <istream>
#include <string>
#include <vector>

#include "sobel5_b200/core.hpp"

namespace sobel5 {

/// Integer BT.601 luma, full range: (77 R + 150 G + 29 B + 128) >> 8
/// (image_io.hpp:20-22).
inline std::uint8_t luma_bt601(int r, int g, int b) {
    return static_cast<std::uint8_t>((77 * r + 150 * g + 29 * b + 128) >> 8);
}

namespace detail {

// ---- PGM ---------------------------------------------------------------------

/// One decimal header value after whitespace and '#' comment lines.
inline int pgm_header_int(std::istream& in) {
    for (;;) {
        const int c = in.peek();
        if (c == EOF) throw CorruptFile("truncated PGM header");
        if (c == '#') {
            std::string skip;
            std::getline(in, skip);
        } else if (std::isspace(c)) {
            in.get();
        } else {
            break;
        }
    }
    int v = 0;
    if (!(in >> v)) throw CorruptFile("malformed PGM header");
    return v;
}

inline GrayPlane load_pgm(std::istream& in, bool binary, const std::string& path) {
    const int w = pgm_header_int(in);
    const int h = pgm_header_int(in);
    const int maxval = pgm_header_int(in);
    if (w <= 0 || h <= 0) throw CorruptFile("bad PGM dimensions in " + path);
    if (maxval != 255)
        throw UnsupportedFormat("PGM maxval " + std::to_string(maxval) + " in " + path +
                                ", only 255 is supported");
    GrayPlane img(w, h);
    auto& px = img.data();
    if (binary) {
        in.get();  // the single whitespace byte that ends the header
        in.read(reinterpret_cast<char*>(px.data()), static_cast<std::streamsize>(px.size()));
        if (static_cast<std::size_t>(in.gcount()) != px.size())
            throw CorruptFile("truncated PGM pixel data in " + path);
        return img;
    }
    for (std::size_t i = 0; i < px.size(); ++i) {
        int v = 0;
        if (!(in >> v)) throw CorruptFile("truncated PGM pixel data in " + path);
        if (v < 0 || v > maxval)
            throw CorruptFile("PGM sample " + std::to_string(v) + " out of range in " + path);
        px[i] = static_cast<std::uint8_t>(v);
    }
    return img;
}

inline void save_pgm(const GrayPlane& img, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot write " + path);
    out << "P5\n" << img.width() << ' ' << img.height() << "\n255\n";
    out.write(reinterpret_cast<const char*>(img.data().data()),
              static_cast<std::streamsize>(img.size()));
    if (!out) throw IoError("short write to " + path);
}

// ---- PNG ---------------------------------------------------------------------

constexpr std::uint8_t kPngSig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
constexpr std::uint32_t kPngMaxDim = 1000000;  // libpng's default user limit

struct PngFail {};  // a decode error libpng would raise (-> CorruptFile)

inline std::uint32_t be32(const std::uint8_t* p) {
    return (std::uint32_t{p[0]} << 24) | (std::uint32_t{p[1]} << 16) | (std::uint32_t{p[2]} << 8) | p[3];
}

inline int paeth(int a, int b, int c) {
    const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
    return pa <= pb && pa <= pc ? a : pb <= pc ? b : c;
}

/// Reverses one row's filter in place (bpp bytes per pixel; prev = the
/// previous reconstructed row of the same pass, or nullptr for the first).
inline void png_unfilter(int type, std::uint8_t* row, const std::uint8_t* prev, std::size_t n, int bpp) {
    switch (type) {
        case 0: return;
        case 1:
            for (std::size_t i = bpp; i < n; ++i) row[i] = static_cast<std::uint8_t>(row[i] + row[i - bpp]);
            return;
        case 2:
            if (prev)
                for (std::size_t i = 0; i < n; ++i) row[i] = static_cast<std::uint8_t>(row[i] + prev[i]);
            return;
        case 3:
            for (std::size_t i = 0; i < n; ++i) {
                const int a = i >= static_cast<std::size_t>(bpp) ? row[i - bpp] : 0, b = prev ? prev[i] : 0;
                row[i] = static_cast<std::uint8_t>(row[i] + ((a + b) >> 1));
            }
            return;
        case 4:
            for (std::size_t i = 0; i < n; ++i) {
                const bool l = i >= static_cast<std::size_t>(bpp);
                const int a = l ? row[i - bpp] : 0, b = prev ? prev[i] : 0, c = l && prev ? prev[i - bpp] : 0;
                row[i] = static_cast<std::uint8_t>(row[i] + paeth(a, b, c));
            }
            return;
        default: throw PngFail{};  // "bad adaptive filter value"
    }
}

struct PngImage {
    std::uint32_t w = 0, h = 0;
    int bit_depth = 0, color_type = 0, interlace = 0;
};

/// The chunk stream up to IEND: IHDR validated as png_read_info does, the
/// IDAT payload concatenated.  Throws PngFail on what libpng rejects;
/// in_image tells whether the first IDAT had been reached (png_read_info
/// returns there, and the reference checks depth and colour type before
/// anything after it is read).
inline void png_parse(const std::vector<std::uint8_t>& f, PngImage& im, std::vector<std::uint8_t>& idat,
                      bool& in_image) {
    std::size_t o = 8;
    bool ihdr = false, iend = false;
    while (!iend) {
        if (f.size() - o < 8) throw PngFail{};  // the file ends before IEND
        const std::uint32_t len = be32(&f[o]);
        const std::uint8_t* type = &f[o + 4];
        if (ihdr && std::memcmp(type, "IDAT", 4) == 0) in_image = true;
        if (len > 0x7fffffffu || f.size() - o < 12 || f.size() - o - 12 < len) throw PngFail{};
        const std::uint8_t* data = &f[o + 8];
        const bool critical = !(type[0] & 0x20);
        const std::uint32_t crc = static_cast<std::uint32_t>(
            crc32(crc32(0L, type, 4), data, static_cast<uInt>(len)));
        const bool crc_ok = crc == be32(data + len);
        o += 12 + static_cast<std::size_t>(len);
        for (int i = 0; i < 4; ++i)
            if (!std::isalpha(type[i])) throw PngFail{};  // invalid chunk type
        if (!crc_ok) {
            if (critical) throw PngFail{};  // CRC error in a critical chunk
            continue;                       // ancillary: discarded (a libpng warning)
        }
        if (std::memcmp(type, "IHDR", 4) == 0) {
            if (ihdr || len != 13) throw PngFail{};
            ihdr = true;
            im.w = be32(data);
            im.h = be32(data + 4);
            im.bit_depth = data[8];
            im.color_type = data[9];
            im.interlace = data[12];
            if (im.w == 0 || im.h == 0 || im.w > kPngMaxDim || im.h > kPngMaxDim) throw PngFail{};
            const int d = im.bit_depth;
            bool ok = false;
            switch (im.color_type) {
                case 0: ok = d == 1 || d == 2 || d == 4 || d == 8 || d == 16; break;
                case 3: ok = d == 1 || d == 2 || d == 4 || d == 8; break;
                case 2: case 4: case 6: ok = d == 8 || d == 16; break;
                default: ok = false;
            }
            if (!ok || data[10] != 0 || data[11] != 0 || im.interlace > 1) throw PngFail{};
            continue;
        }
        if (!ihdr) throw PngFail{};  // IHDR must come first
        if (std::memcmp(type, "IDAT", 4) == 0) {
            in_image = true;
            idat.insert(idat.end(), data, data + len);
        } else if (std::memcmp(type, "IEND", 4) == 0) {
            iend = true;
        } else if (std::memcmp(type, "PLTE", 4) == 0) {
            if (im.color_type == 3 && (len == 0 || len % 3 != 0 || len > 768)) throw PngFail{};
        } else if (critical) {
            throw PngFail{};  // unknown critical chunk
        }
    }
    if (idat.empty()) throw PngFail{};  // no image data
}

/// Decodes 8-bit gray / RGB / RGBA image data (interlaced or not) into
/// interleaved pixels, w * h * ch bytes.
inline std::vector<std::uint8_t> png_decode_pixels(const PngImage& im, int ch,
                                                   const std::vector<std::uint8_t>& idat) {
    struct Pass {
        int x0, y0, dx, dy;
    };
    static constexpr Pass kAdam7[7] = {{0, 0, 8, 8}, {4, 0, 8, 8}, {0, 4, 4, 8}, {2, 0, 4, 4},
                                       {0, 2, 2, 4}, {1, 0, 2, 2}, {0, 1, 1, 2}};
    const Pass kFlat[1] = {{0, 0, 1, 1}};
    const Pass* passes = im.interlace ? kAdam7 : kFlat;
    const int n_pass = im.interlace ? 7 : 1;
    const std::size_t W = im.w, H = im.h;
    std::size_t need = 0;
    for (int p = 0; p < n_pass; ++p) {
        const std::size_t pw = (W + passes[p].dx - 1 - passes[p].x0) / passes[p].dx;
        const std::size_t ph = (H + passes[p].dy - 1 - passes[p].y0) / passes[p].dy;
        if (W > static_cast<std::size_t>(passes[p].x0) && H > static_cast<std::size_t>(passes[p].y0))
            need += ph * (1 + pw * ch);
    }
    std::vector<std::uint8_t> raw(need);
    z_stream zs{};
    if (inflateInit(&zs) != Z_OK) throw PngFail{};
    zs.next_in = const_cast<Bytef*>(idat.data());
    zs.avail_in = static_cast<uInt>(idat.size());
    zs.next_out = raw.data();
    zs.avail_out = static_cast<uInt>(raw.size());
    int r = Z_OK;
    while (zs.avail_out > 0 && r == Z_OK) r = inflate(&zs, Z_NO_FLUSH);
    inflateEnd(&zs);
    // all rows present is what counts; a stream that ended early, or broke
    // before the last row, is missing image data.  Trailing bytes or a bad
    // checksum after the last row are libpng warnings.
    if (zs.avail_out != 0) throw PngFail{};

    std::vector<std::uint8_t> out(W * H * ch);
    std::size_t off = 0;
    for (int p = 0; p < n_pass; ++p) {
        const Pass& ps = passes[p];
        if (W <= static_cast<std::size_t>(ps.x0) || H <= static_cast<std::size_t>(ps.y0)) continue;
        const std::size_t pw = (W + ps.dx - 1 - ps.x0) / ps.dx, ph = (H + ps.dy - 1 - ps.y0) / ps.dy;
        const std::size_t rb = pw * ch;
        const std::uint8_t* prev = nullptr;
        for (std::size_t y = 0; y < ph; ++y) {
            std::uint8_t* row = raw.data() + off + 1;
            png_unfilter(raw[off], row, prev, rb, ch);
            const std::size_t oy = ps.y0 + y * ps.dy;
            for (std::size_t x = 0; x < pw; ++x)
                std::memcpy(&out[(oy * W + ps.x0 + x * ps.dx) * ch], row + x * ch, ch);
            prev = row;
            off += 1 + rb;
        }
    }
    return out;
}

inline std::vector<std::uint8_t> read_file(const std::string& path) {
    std::FILE* fp = std::fopen(path.c_str(), "rb");
    if (!fp) throw IoError("cannot open " + path);
    std::vector<std::uint8_t> f;
    std::uint8_t buf[1 << 16];
    for (std::size_t n; (n = std::fread(buf, 1, sizeof buf, fp)) > 0;) f.insert(f.end(), buf, buf + n);
    std::fclose(fp);
    return f;
}

inline GrayPlane load_png(const std::string& path) {
    const std::vector<std::uint8_t> f = read_file(path);
    if (f.size() < 8 || std::memcmp(f.data(), kPngSig, 8) != 0)
        throw CorruptFile("bad PNG signature in " + path);
    PngImage im;
    std::vector<std::uint8_t> idat;
    bool in_image = false, broken = false;
    try {
        png_parse(f, im, idat, in_image);
    } catch (const PngFail&) {
        // before the first IDAT: png_read_info fails; after it, the
        // reference checks depth and colour type first (image_io.hpp:105-117)
        if (!in_image) throw CorruptFile("libpng failed to decode " + path);
        broken = true;
    }
    if (im.bit_depth != 8)
        throw UnsupportedFormat("PNG bit depth " + std::to_string(im.bit_depth) + " in " + path +
                                ", only 8 is supported");
    int ch = 0;
    switch (im.color_type) {
        case 0: ch = 1; break;
        case 2: ch = 3; break;
        case 6: ch = 4; break;
        default:
            throw UnsupportedFormat("PNG color type " + std::to_string(im.color_type) + " in " + path +
                                    ", need gray, RGB or RGBA");
    }
    if (broken) throw CorruptFile("libpng failed to decode " + path);
    std::vector<std::uint8_t> px;
    try {
        px = png_decode_pixels(im, ch, idat);
    } catch (const PngFail&) {
        throw CorruptFile("libpng failed to decode " + path);
    }
    GrayPlane img(static_cast<int>(im.w), static_cast<int>(im.h));
    auto& g = img.data();
    if (ch == 1) {
        std::copy(px.begin(), px.end(), g.begin());
    } else {
        for (std::size_t i = 0; i < g.size(); ++i) {
            const std::uint8_t* p = px.data() + i * ch;
            g[i] = luma_bt601(p[0], p[1], p[2]);
        }
    }
    return img;
}

inline void png_put32(std::vector<std::uint8_t>& o, std::uint32_t v) {
    for (int s = 24; s >= 0; s -= 8) o.push_back(static_cast<std::uint8_t>(v >> s));
}
inline void png_chunk(std::vector<std::uint8_t>& o, const char* type, const std::uint8_t* d, std::size_t n) {
    png_put32(o, static_cast<std::uint32_t>(n));
    const std::size_t t = o.size();
    o.insert(o.end(), type, type + 4);
    if (n) o.insert(o.end(), d, d + n);
    png_put32(o, static_cast<std::uint32_t>(crc32(0L, o.data() + t, static_cast<uInt>(n + 4))));
}

/// The filtered scanlines of an 8-bit gray image: per row, the filter with
/// the minimum sum of absolute signed residuals (libpng's default
/// heuristic; ties go to the earlier of None, Sub, Up, Average, Paeth).
inline std::vector<std::uint8_t> png_filter_gray(const GrayPlane& img) {
    const std::size_t w = img.width(), h = img.height();
    std::vector<std::uint8_t> out;
    out.reserve(h * (w + 1));
    std::array<std::vector<std::uint8_t>, 5> cand;
    for (auto& c : cand) c.resize(w);
    for (std::size_t y = 0; y < h; ++y) {
        const std::uint8_t* row = img.data().data() + y * w;
        const std::uint8_t* up = y ? row - w : nullptr;
        for (std::size_t i = 0; i < w; ++i) {
            const int a = i ? row[i - 1] : 0, b = up ? up[i] : 0, c = i && up ? up[i - 1] : 0;
            cand[0][i] = row[i];
            cand[1][i] = static_cast<std::uint8_t>(row[i] - a);
            cand[2][i] = static_cast<std::uint8_t>(row[i] - b);
            cand[3][i] = static_cast<std::uint8_t>(row[i] - ((a + b) >> 1));
            cand[4][i] = static_cast<std::uint8_t>(row[i] - paeth(a, b, c));
        }
        int best = 0;
        std::uint64_t best_sum = ~std::uint64_t{0};
        for (int f = 0; f < 5; ++f) {
            std::uint64_t s = 0;
            for (std::size_t i = 0; i < w; ++i) s += cand[f][i] < 128 ? cand[f][i] : 256 - cand[f][i];
            if (s < best_sum) {
                best_sum = s;
                best = f;
            }
        }
        out.push_back(static_cast<std::uint8_t>(best));
        out.insert(out.end(), cand[best].begin(), cand[best].end());
    }
    return out;
}

inline void save_png_gray(const GrayPlane& img, const std::string& path) {
    std::FILE* fp = std::fopen(path.c_str(), "wb");
    if (!fp) throw IoError("cannot write " + path);
    std::vector<std::uint8_t> o(kPngSig, kPngSig + 8);
    std::uint8_t ihdr[13];
    const std::uint32_t w = static_cast<std::uint32_t>(img.width()), h = static_cast<std::uint32_t>(img.height());
    for (int i = 0; i < 4; ++i) {
        ihdr[i] = static_cast<std::uint8_t>(w >> (24 - 8 * i));
        ihdr[4 + i] = static_cast<std::uint8_t>(h >> (24 - 8 * i));
    }
    ihdr[8] = 8;  // bit depth
    ihdr[9] = 0;  // gray
    ihdr[10] = ihdr[11] = ihdr[12] = 0;
    png_chunk(o, "IHDR", ihdr, 13);
    const std::vector<std::uint8_t> raw = png_filter_gray(img);
    uLongf zn = compressBound(static_cast<uLong>(raw.size()));
    std::vector<std::uint8_t> z(zn);
    bool ok = compress2(z.data(), &zn, raw.data(), static_cast<uLong>(raw.size()), Z_DEFAULT_COMPRESSION) == Z_OK;
    if (ok) {
        constexpr std::size_t kIdat = 8192;  // libpng's default IDAT size
        for (std::size_t a = 0; a < zn; a += kIdat) png_chunk(o, "IDAT", z.data() + a, std::min(kIdat, zn - a));
        png_chunk(o, "IEND", nullptr, 0);
        ok = std::fwrite(o.data(), 1, o.size(), fp) == o.size();
    }
    ok = std::fclose(fp) == 0 && ok;
    if (!ok) throw IoError("libpng failed to encode " + path);
}

inline bool has_suffix(const std::string& s, const std::string& suffix) {
    return s.size() >= suffix.size() &&
           std::equal(suffix.rbegin(), suffix.rend(), s.rbegin(), [](char a, char b) {
               return std::tolower(static_cast<unsigned char>(b)) == a;
           });
}

}  // namespace detail

/// An image as 8-bit grayscale; the format is sniffed from the leading bytes
/// (PGM P2 / P5 or PNG), colour PNG reduced with integer BT.601 luma
/// (image_io.hpp:201-213).
inline GrayPlane load_gray(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path);
    const int m0 = in.get();
    const int m1 = in.get();
    if (m0 == 'P' && (m1 == '2' || m1 == '5')) return detail::load_pgm(in, m1 == '5', path);
    if (m0 == 0x89 && m1 == 'P') {
        in.close();
        return detail::load_png(path);
    }
    throw UnsupportedFormat("unrecognized image format in " + path);
}

/// Writes an 8-bit plane; the extension picks PGM (P5) or PNG
/// (image_io.hpp:216-223).
inline void save_gray(const GrayPlane& img, const std::string& path) {
    if (detail::has_suffix(path, ".pgm"))
        detail::save_pgm(img, path);
    else if (detail::has_suffix(path, ".png"))
        detail::save_png_gray(img, path);
    else
        throw UnsupportedExtension("cannot infer image format from " + path);
}

}  // namespace sobel5
