/*
 * sobel5_oracle.c -- CPU restatement of the reference 4-direction 5x5 Sobel
 * path.  TEST INFRASTRUCTURE ONLY (see sobel5_oracle.h): the checker for the
 * CUDA path and the CPU timing arm, never part of the product.
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to the reference's proj/include/sobel5/.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared (oracle/Makefile).
 * -ffp-contract=off keeps the magnitude's (mul, add) sequence unfused, as the
 * reference's -O3 build without -march does (hard part 3).
 */
#include "sobel5_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- filter algebra ---------------------------------------------------- */

/* materialize_exact() for integer parameters: filter_algebra.hpp:82-134.
 * X: a*col(1,n,m,n,1) x row(-1,-b,0,b,1)           (:92-98)
 * Y: a*col(-1,-b,0,b,1) x row(1,n,m,n,1)           (:100-106)
 * D, DT: the explicit matrices                     (:108-131) */
void oracle_materialize(int64_t a, int64_t b, int64_t m, int64_t n, int dir, int32_t k[25]) {
    const int64_t nb = n * b, mb = m * b;
    int64_t w[25];
    if (dir == 0 || dir == 1) {
        const int64_t smooth[5] = {1, n, m, n, 1};
        const int64_t deriv[5] = {-1, -b, 0, b, 1};
        for (int i = 0; i < 5; ++i)
            for (int j = 0; j < 5; ++j)
                w[i * 5 + j] = dir == 0 ? smooth[i] * deriv[j] : deriv[i] * smooth[j];
    } else if (dir == 2) {
        const int64_t d[25] = {-m, -n,  -1,  -b, 0,  -n, -mb, -nb, 0,  b,  -1, -nb, 0,
                               nb, 1,  -b,  0,  nb, mb, n,   0,   b, 1, n,  m};
        memcpy(w, d, sizeof w);
    } else {
        const int64_t d[25] = {0, -b, -1,  -n, -m, b,  0,  -nb, -mb, -n, 1, nb, 0,
                               -nb, -1, n, mb, nb, 0,  -b, m,  n,   1,   b, 0};
        memcpy(w, d, sizeof w);
    }
    for (int i = 0; i < 25; ++i) k[i] = (int32_t)(a * w[i]);
}

/* make_stream_taps(): pipeline.hpp:75-107. */
void oracle_make_stream_taps(int64_t a64, int64_t b64, int64_t m64, int64_t n64, oracle_taps* t) {
    const int32_t a = (int32_t)a64, b = (int32_t)b64, m = (int32_t)m64, n = (int32_t)n64;
    const int32_t f[5] = {-1, -b, 0, b, 1};
    const int32_t h[5] = {1, n, m, n, 1};
    const int32_t k0[5] = {-a * m, -a * (n + b), -2 * a, -a * (n + b), -a * m};
    const int32_t k1[5] = {a * (b - n), -a * m * b, -2 * a * n * b, -a * m * b, a * (b - n)};
    const int32_t gx_v[5] = {a, a * n, a * m, a * n, a};
    const int32_t gy_v[5] = {-a, -a * b, 0, a * b, a};
    const int32_t gdm_f[5] = {a * m, a * (n + b), 2 * a, a * (n + b), a * m};
    const int32_t gdm_d[5] = {a * (m * b + b - n), a * (n * b + b * b - m * b),
                              a * (2 * b - 2 * n * b), a * (n * b + b * b - m * b),
                              a * (m * b + b - n)};
    t->a = a;
    memcpy(t->f, f, sizeof f);
    memcpy(t->h, h, sizeof h);
    memcpy(t->k0, k0, sizeof k0);
    memcpy(t->k1, k1, sizeof k1);
    memcpy(t->gx_v, gx_v, sizeof gx_v);
    memcpy(t->gy_v, gy_v, sizeof gy_v);
    memcpy(t->gdm_f, gdm_f, sizeof gdm_f);
    memcpy(t->gdm_d, gdm_d, sizeof gdm_d);

    /* wide_vagg bound: pipeline.hpp:94-105 */
    int64_t sf = 0, sh = 0, sgx = 0, sgy = 0, sdf = 0, sdd = 0;
    for (int i = 0; i < 5; ++i) {
        sf += llabs(f[i]);
        sh += llabs(h[i]);
        sgx += llabs(gx_v[i]);
        sgy += llabs(gy_v[i]);
        sdf += llabs(gdm_f[i]);
        sdd += llabs(gdm_d[i]);
    }
    const int64_t max_f_row = 255 * sf, max_h_row = 255 * sh;
    int64_t bound = sgx * max_f_row;
    if (sgy * max_h_row > bound) bound = sgy * max_h_row;
    if (sdf * max_f_row + sdd * 510 > bound) bound = sdf * max_f_row + sdd * 510;
    t->wide_vagg = bound > INT32_MAX;
}

/* ---- oracle.hpp -------------------------------------------------------- */

/* conv2d_valid(GrayPlane, Kernel5): oracle.hpp:19-33. */
int oracle_conv2d_valid(const uint8_t* img, int w, int h, const int32_t k[25], int32_t* out) {
    if (w < 5 || h < 5) return 1;
    const int ow = w - 4, oh = h - 4;
    for (int y = 0; y < oh; ++y)
        for (int x = 0; x < ow; ++x) {
            int64_t acc = 0;
            for (int i = 0; i < 5; ++i)
                for (int j = 0; j < 5; ++j)
                    acc += (int64_t)k[i * 5 + j] * img[(size_t)(y + i) * w + x + j];
            out[(size_t)y * ow + x] = (int32_t)acc;
        }
    return 0;
}

/* conv2d_valid(GrayPlane, Kernel3): oracle.hpp:35-49 (the same window sum
 * at radius 1). */
int oracle_conv2d_valid3(const uint8_t* img, int w, int h, const int32_t k[9], int32_t* out) {
    if (w < 3 || h < 3) return 1;
    const int ow = w - 2, oh = h - 2;
    for (int y = 0; y < oh; ++y)
        for (int x = 0; x < ow; ++x) {
            int64_t acc = 0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j)
                    acc += (int64_t)k[i * 3 + j] * img[(size_t)(y + i) * w + x + j];
            out[(size_t)y * ow + x] = (int32_t)acc;
        }
    return 0;
}

/* Magnitude, oracle.hpp:89-96 and pipeline.hpp:401-407: left-to-right sum
 * of products in double, then sqrt. */
static double magnitude(int32_t gx, int32_t gy, int32_t gd, int32_t gdt) {
    const double x = gx, y = gy, d = gd, t = gdt;
    double s = x * x;
    s = s + y * y;
    s = s + d * d;
    s = s + t * t;
    return sqrt(s);
}

/* sobel5_4d(): oracle.hpp:82-98.  Planes the caller did not ask for are
 * still computed (into scratch) when g is requested. */
int oracle_sobel5_4d(const uint8_t* img, int w, int h, int64_t a, int64_t b, int64_t m,
                     int64_t n, int32_t* gx, int32_t* gy, int32_t* gd, int32_t* gdt,
                     double* g) {
    if (w < 5 || h < 5) return 1;
    const size_t count = (size_t)(w - 4) * (size_t)(h - 4);
    int32_t* planes[4] = {gx, gy, gd, gdt};
    int32_t* owned[4] = {NULL, NULL, NULL, NULL};
    int32_t k[25];
    for (int dir = 0; dir < 4; ++dir) {
        if (!planes[dir]) {
            if (!g) continue;
            owned[dir] = (int32_t*)malloc(count * sizeof(int32_t));
            if (!owned[dir]) return 2;
            planes[dir] = owned[dir];
        }
        oracle_materialize(a, b, m, n, dir, k);
        oracle_conv2d_valid(img, w, h, k, planes[dir]);
    }
    if (g)
        for (size_t i = 0; i < count; ++i)
            g[i] = magnitude(planes[0][i], planes[1][i], planes[2][i], planes[3][i]);
    for (int dir = 0; dir < 4; ++dir) free(owned[dir]);
    return 0;
}

/* ---- run_stream arithmetic contract ------------------------------------- */

/* row_conv5 (pipeline.hpp:117-122) at one position, wrapping mod 2^32. */
static uint32_t conv5(const uint8_t* p, const int32_t taps[5]) {
    uint32_t s = 0;
    for (int j = 0; j < 5; ++j) s += (uint32_t)taps[j] * (uint32_t)p[j];
    return s;
}

int oracle_run_stream(const uint8_t* img, int w, int h, const oracle_taps* t, int32_t* gx,
                      int32_t* gy, int32_t* gd, int32_t* gdt, double* g, int32_t* bad_sum,
                      int32_t* bad_diff) {
    /* run_stream validation: pipeline.hpp:454-456 */
    if (w < 5 || h < 5) return 1;
    const int ow = w - 4, oh = h - 4;
    int status = 0;
    for (int y = 0; y < oh; ++y)
        for (int x = 0; x < ow; ++x) {
            uint32_t ax = 0, ay = 0, am = 0, ap;
            uint32_t k0[5], k1[5];
            for (int i = 0; i < 5; ++i) {
                const uint8_t* p = img + (size_t)(y + i) * w + x;
                const uint32_t F = conv5(p, t->f);                    /* :327 */
                const uint32_t H = conv5(p, t->h);                    /* :328 */
                const uint32_t D = (uint32_t)p[3] - (uint32_t)p[1];   /* :124-127 */
                ax += (uint32_t)t->gx_v[i] * F;                       /* :389/:393 */
                ay += (uint32_t)t->gy_v[i] * H;                       /* :390/:394 */
                am += (uint32_t)t->gdm_f[i] * F - (uint32_t)t->gdm_d[i] * D; /* :182-186 */
                k0[i] = conv5(p, t->k0);                              /* :336 */
                k1[i] = conv5(p, t->k1);                              /* :341 */
            }
            /* Eq. 15 with the bank signs (+,+,-,-): pipeline.hpp:152-164 */
            ap = k0[0] + k1[1] - k1[3] - k0[4];
            const int32_t P = (int32_t)ap, M = (int32_t)am;
            const int32_t sum = (int32_t)((uint32_t)P + (uint32_t)M);
            /* recover_diag: pipeline.hpp:268-273 */
            if ((sum & 1) != 0) {
                if (status == 0) {
                    if (bad_sum) *bad_sum = P;
                    if (bad_diff) *bad_diff = M;
                }
                status = 3;
                continue;
            }
            const int32_t vd = sum / 2;
            const int32_t vdt = (int32_t)((uint32_t)P - (uint32_t)M) / 2;
            const size_t o = (size_t)y * ow + x;
            if (gx) gx[o] = (int32_t)ax;
            if (gy) gy[o] = (int32_t)ay;
            if (gd) gd[o] = vd;
            if (gdt) gdt[o] = vdt;
            if (g) g[o] = magnitude((int32_t)ax, (int32_t)ay, vd, vdt);
        }
    return status;
}

/* detail::quantize(..., clamp_abs): image_io.hpp:235-240. */
void oracle_clamp_abs_f64(const double* g, size_t count, uint8_t* out) {
    for (size_t i = 0; i < count; ++i) {
        const double v = fabs(g[i]);
        const double r = round(v);
        out[i] = (uint8_t)(r < 255.0 ? r : 255.0);
    }
}

/* splitmix64 + synth_random: synth.hpp:11-35. */
void oracle_synth_random(uint8_t* img, int w, int h, uint64_t seed) {
    uint64_t state = seed, word = 0;
    int have = 0;
    const size_t count = (size_t)w * (size_t)h;
    for (size_t i = 0; i < count; ++i) {
        if (have == 0) {
            state += 0x9E3779B97F4A7C15ULL;
            uint64_t z = state;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            word = z ^ (z >> 31);
            have = 8;
        }
        img[i] = (uint8_t)(word & 0xFF);
        word >>= 8;
        --have;
    }
}

/* Walks run_strip's schedule (pipeline.hpp:304-414) for the tallies. */
static uint64_t nonzero(const int32_t taps[5]) { /* pipeline.hpp:111-115 */
    uint64_t c = 0;
    for (int i = 0; i < 5; ++i) c += taps[i] != 0;
    return c;
}

void oracle_stream_counters(int h, const int* strip_out_w, int n_strips, const oracle_taps* t,
                            int prefetch, oracle_counters* c) {
    memset(c, 0, sizeof *c);
    const uint64_t nzf = nonzero(t->f), nzh = nonzero(t->h), nzk0 = nonzero(t->k0),
                   nzk1 = nonzero(t->k1);
    const uint64_t center = nonzero(t->gx_v) + nonzero(t->gy_v) + 4 + nonzero(t->gdm_f) +
                            nonzero(t->gdm_d);
    for (int s = 0; s < n_strips; ++s) {
        const uint64_t w = (uint64_t)strip_out_w[s];
#define HPASS()                         \
    do {                                \
        c->row_conv5_f += 1;            \
        c->row_conv5_h += 1;            \
        c->row_diff += 1;               \
        c->mac += (nzf + nzh + 2) * w;  \
    } while (0)
#define BANK_K0()                \
    do {                         \
        c->row_conv5_k0 += 1;    \
        c->mac += nzk0 * w;      \
    } while (0)
#define BANK_K1()                \
    do {                         \
        c->row_conv5_k1 += 1;    \
        c->mac += nzk1 * w;      \
    } while (0)
        for (int u = 0; u < 5; ++u) HPASS(); /* :347 */
        BANK_K0();                           /* :348-352 */
        BANK_K1();
        BANK_K1();
        BANK_K1();
        BANK_K0();
        const int64_t last = h - 3;
        for (int64_t v = 2; v <= last; ++v) {
            if (prefetch) { /* :362-369 */
                if (v + 3 <= h - 1) {
                    HPASS();
                    BANK_K0();
                }
                if (v > 2) BANK_K0();
            } else if (v > 2) { /* :370-374 */
                HPASS();
                BANK_K0();
                BANK_K0();
            }
            c->mac += center * w;    /* :399 */
            if (v < last) BANK_K1(); /* :411 */
        }
#undef HPASS
#undef BANK_K0
#undef BANK_K1
    }
}

uint64_t oracle_fnv1a64(const void* data, size_t bytes) {
    const uint8_t* p = (const uint8_t*)data;
    uint64_t hsh = 1469598103934665603ULL;
    for (size_t i = 0; i < bytes; ++i) {
        hsh ^= p[i];
        hsh *= 1099511628211ULL;
    }
    return hsh;
}

/* ---- detect-path pieces -------------------- */

static int clampi(int v, int lo, int hi) { return v < lo ? lo : v > hi ? hi : v; }

/* pad_replicate (image_io.hpp:279-291): (w+2r) x (h+2r), every border pixel
 * the nearest edge pixel (std::clamp of both coordinates). Returns 0,
 * 20 (EmptyPlane, :280) or 19 (DimMismatch for r < 0, :281). */
int oracle_pad_replicate(const uint8_t* img, int w, int h, int r, uint8_t* out) {
    if (w <= 0 || h <= 0) return 20;
    if (r < 0) return 19;
    const int pw = w + 2 * r, ph = h + 2 * r;
    for (int y = 0; y < ph; ++y) {
        const int sy = clampi(y - r, 0, h - 1);
        for (int x = 0; x < pw; ++x) out[(size_t)y * pw + x] = img[(size_t)sy * w + clampi(x - r, 0, w - 1)];
    }
    return 0;
}

/* detail::quantize(plane, normalize) (image_io.hpp:242-255): lo/hi by a
 * sequential std::min/std::max scan from element 0, then
 * lround((v - lo) * 255.0 / span) in double, 0 when span <= 0. */
static void normalize_doubles(const double* v, size_t n, uint8_t* out) {
    if (n == 0) return;
    double lo = v[0], hi = v[0];
    for (size_t i = 1; i < n; ++i) {
        lo = v[i] < lo ? v[i] : lo; /* std::min(lo, v): returns lo unless v < lo */
        hi = hi < v[i] ? v[i] : hi; /* std::max(hi, v): returns hi unless hi < v */
    }
    const double span = hi - lo;
    for (size_t i = 0; i < n; ++i) {
        const double mapped = span > 0 ? (v[i] - lo) * 255.0 / span : 0.0;
        out[i] = (uint8_t)lround(mapped);
    }
}

void oracle_normalize_f64(const double* v, size_t n, uint8_t* out) { normalize_doubles(v, n, out); }

void oracle_normalize_i32(const int32_t* v, size_t n, uint8_t* out) {
    /* quantize<int32_t> converts each element with static_cast<double>
     * (image_io.hpp:243-249); every int32 is exact in double */
    if (n == 0) return;
    double* d = (double*)malloc(n * sizeof(double));
    for (size_t i = 0; i < n; ++i) d[i] = (double)v[i];
    normalize_doubles(d, n, out);
    free(d);
}

/* quantize<int32_t>(plane, clamp_abs) (image_io.hpp:235-240). */
void oracle_clamp_abs_i32(const int32_t* v, size_t n, uint8_t* out) {
    for (size_t i = 0; i < n; ++i) {
        const double a = fabs((double)v[i]);
        const double r = round(a);
        out[i] = (uint8_t)(r < 255.0 ? r : 255.0);
    }
}

/* sobel3_2d (oracle.hpp:58-70) with kernel3_x / kernel3_y
 * (filter_algebra.hpp:33-39), valid mode, int64 accumulation cast to
 * int32 (conv2d_valid, oracle.hpp:35-48), g = sqrt(gx*gx + gy*gy). */
int oracle_sobel3_2d(const uint8_t* img, int w, int h, int32_t* gx, int32_t* gy, double* g) {
    static const int32_t kx[3][3] = {{-1, 0, 1}, {-2, 0, 2}, {-1, 0, 1}};
    static const int32_t ky[3][3] = {{-1, -2, -1}, {0, 0, 0}, {1, 2, 1}};
    if (w < 3 || h < 3) return 1;
    const int ow = w - 2, oh = h - 2;
    for (int y = 0; y < oh; ++y)
        for (int x = 0; x < ow; ++x) {
            int64_t ax = 0, ay = 0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    const int64_t p = img[(size_t)(y + i) * w + x + j];
                    ax += kx[i][j] * p;
                    ay += ky[i][j] * p;
                }
            const size_t o = (size_t)y * ow + x;
            if (gx) gx[o] = (int32_t)ax;
            if (gy) gy[o] = (int32_t)ay;
            if (g) {
                const double dx = (double)(int32_t)ax, dy = (double)(int32_t)ay;
                g[o] = sqrt(dx * dx + dy * dy);
            }
        }
    return 0;
}

/* OpCounters of run_stream_3x3 (pipeline.hpp:488-547): per strip, one hpass
 * (F and H row_conv3, mac += 5w) per primed row (3) and per later centre,
 * and mac += 5w per centre. */
void oracle_stream3_counters(int h, const int* strip_out_w, int n_strips, int prefetch,
                             oracle_counters* c) {
    memset(c, 0, sizeof *c);
    for (int s = 0; s < n_strips; ++s) {
        const uint64_t w = (uint64_t)strip_out_w[s];
#define HPASS3()                \
    do {                        \
        c->row_conv3_f += 1;    \
        c->row_conv3_h += 1;    \
        c->mac += 5 * w;        \
    } while (0)
        for (int u = 0; u < 3; ++u) HPASS3(); /* :514 */
        for (int64_t v = 1; v <= h - 2; ++v) {
            if (prefetch) { /* :518-519 */
                if (v + 2 <= h - 1) HPASS3();
            } else if (v > 1) { /* :520-522 */
                HPASS3();
            }
            c->mac += 5 * w; /* :545 */
        }
#undef HPASS3
    }
}
