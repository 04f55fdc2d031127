// sobel5_stream.cuh -- the fused streaming 4-direction 5x5 Sobel kernel for
// sm_100a (B200).
//
// One kernel replaces the reference's whole per-strip schedule
// (pipeline.hpp:304-414): horizontal passes F/H/D/K0/K1 (row_conv5 :117-122,
// row_diff :124-127), vertical aggregation of gx, gy, Gd- and Gd+ (vagg5
// :136-150, vagg_gd_minus :166-189, vagg_gd_plus :152-164), exact halving
// (recover_diag :268-282), the double magnitude (:401-407) and, optionally,
// the clamp_abs uint8 edge map (image_io.hpp:235-240) and a float magnitude.
//
// Geometry:
//   * a warp owns 128 consecutive output columns, 4 per lane; a CTA is 4
//     warps side by side (512 columns) and streams a band of `band` output
//     rows top to bottom (band + 4 input rows, the 2r vertical halo).
//   * each lane loads ONE 32-bit word (4 pixels) per input row; the 4 pixels
//     to its right come from lane+1 by __shfl_down_sync (the paper's warp
//     shuffle column sharing); lane 31 loads its right
//     neighbour word itself, so no lane of the warp idles.
//   * instead of a ring of horizontal rows (RowRing, ring.hpp:16-57) the
//     kernel keeps the vertical sums as running accumulators: input row r
//     contributes coefficient i = r - v to the four pending output rows
//     v = r-4 .. r.  That needs 4 quantities x 4 live rows x 4 pixels = 64
//     registers instead of a 5 x 5-quantity ring, and the K_d+ stream needs
//     no bank: each row's K0 and K1 are computed once and folded with their
//     Eq. 14 signs (+K0 at i=0, +K1 at i=1, -K1 at i=3, -K0 at i=4).
//   * all 32-bit arithmetic wraps (unsigned), which reproduces both the
//     reference's int32 path and its int64 "wide_vagg" path followed by the
//     int32 narrowing cast, for ANY caller-supplied taps.
#pragma once

#include <cuda.h>

#include <cstdint>

#include "sobel5_gpu.h"

namespace sobel5_b200 {

constexpr int kWarpCols = 128;          // output columns per warp (4 per lane)
#ifndef SOBEL5_CTA_WARPS
#define SOBEL5_CTA_WARPS 4
#endif
constexpr int kCtaWarps = SOBEL5_CTA_WARPS;  // warps per CTA, side by side
constexpr int kCtaCols = kWarpCols * kCtaWarps;
constexpr int kCtaThreads = 32 * kCtaWarps;
constexpr int kMinCtasPerSm = 16 / kCtaWarps;  // 16 resident warps per SM (<= 128 registers)

enum MagMode : int {
    kMagU32 = 0,  // exact integer sum of squares fits uint32 (host-proven bound)
    kMagF64 = 1,  // general: the reference's ((x*x + y*y) + d*d) + t*t in double
    kMagU64 = 2,  // exact integer sum of squares < 2^53 in uint64 (then double(S) is exact)
};

struct KernelParams {
    // input: three vertical segments (halo above, body, halo below); a plain
    // image is body only.  Rows are addressed in "stacked" coordinates.
    const uint8_t* top;
    const uint8_t* mid;
    const uint8_t* bot;
    int64_t in_pitch;
    int64_t in_frame_stride;
    int top_rows;  // 0 or 2
    int mid_rows;
    int width;     // input columns
    int out_w;     // width - 4
    int out_h;     // total stacked rows - 4
    int band;      // output rows per CTA
    // outputs
    int32_t* gx;
    int32_t* gy;
    int32_t* gd;
    int32_t* gdt;
    double* g;
    float* g32;
    uint8_t* u8;
    int64_t pitch;
    int64_t out_frame_stride;
    sobel5_diag* diag;
    // the launch's first frame / output row in the caller's image (a row
    // chunk, a frame of a stream, a band of a partition): the ParityViolation
    // order key is global, not launch-local
    int diag_frame0;
    int diag_row0;
    int need_mag;
    // detect path: replicate padding, normalize export
    int pad;                     // 1: pad_replicate(img, 2) fused (same-size output)
    sobel5_minmax* minmax;       // per frame: min/max of g (pass 1 of normalize)
    const sobel5_norm_table* norm;  // per frame: normalize thresholds (pass 2)
    int u8_norm;                 // u8 plane = normalize(g) instead of clamp_abs(g)
    uint32_t* s32;               // exact integer g^2 (normalize pass 1 of the detect path)
    // taps (kernel parameter space -> constant-bank operands)
    int32_t f[5], h[5], k0[5], k1[5], gx_v[5], gy_v[5], gdm_f[5], gdm_d[5];
    int tma_load;  // packed plain kernel: band rows bulk-copied into shared memory
    int frames;    // frames of the launch
    int tstore;    // StreamResult by TMA tensor stores (tmap valid)
    int n16;       // gx gy gd gdt as int16 at the int32 pointers (host wire, kOutN16)
    // the same taps as floats for the packed-FP32 kernel (sobel5_f32x2.cuh):
    // f, h, k0, k1, gx_v, gy_v, gdm_f, -gdm_d
    float tf[8][5];
    // StreamResult by TMA tensor stores (kGeomPlainTmaTs): gx, gy, gd, gdt
    // (as uint64 pairs) and g, built on the host (sobel5_tmap.cu)
    alignas(64) CUtensorMap tmap[5];
};

// Compile-time default taps, (a, b, m, n) = (1, 2, 6, 4) (make_stream_taps,
// pipeline.hpp:75-107); used by the specialised instantiation only when the
// host has compared the caller's taps equal to these.
struct DefaultTaps {
    static constexpr int32_t f[5] = {-1, -2, 0, 2, 1};
    static constexpr int32_t h[5] = {1, 4, 6, 4, 1};
    static constexpr int32_t k0[5] = {-6, -6, -2, -6, -6};
    static constexpr int32_t k1[5] = {-2, -12, -16, -12, -2};
    static constexpr int32_t gx_v[5] = {1, 4, 6, 4, 1};
    static constexpr int32_t gy_v[5] = {-1, -2, 0, 2, 1};
    static constexpr int32_t gdm_f[5] = {6, 6, 2, 6, 6};
    static constexpr int32_t gdm_d[5] = {10, 0, -12, 0, 10};
};

// Programmatic dependent launch (PDL): the launchers set
// cudaLaunchAttributeProgrammaticStreamSerialization, so the next kernel in
// the stream may be scheduled once every CTA of this one has started
// (launch_dependents as the first instruction), and this kernel waits for
// its predecessor's completion and memory flush before touching global
// memory (griddepcontrol.wait, before any load or store).  Back-to-back
// frames thus overlap one launch's CTA scheduling with the previous tail.
// Without the attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ParityViolation bookkeeping (recover_diag, pipeline.hpp:268-273).  The
// pair kept is the one the reference reports with workers = 1 -- strips of
// d->strip_w output columns left to right, then rows top to bottom, then
// columns (run_strips_parallel :416-445 walks the strips in order, run_strip
// the rows, recover_diag the columns).  Position key: frame 10 bits, strip
// 16, row 22, column in strip 16, each saturated.
//
// Kept off the row loop's registers: a thread notes its first odd pixel in
// its own shared-memory slot (rare path, no extra live registers in the
// hot loop) and publishes it once at the end of the kernel, where the
// device word {~key, sum, diff} changes by one 16-byte CAS (stored inverted
// so a zeroed word means "none").  Only fault-injected taps produce odd pairs.
struct OddSlot {
    unsigned long long key;  // ~0 = none
    int32_t p, m;
};
__device__ __forceinline__ void odd_init(OddSlot* s) { s[threadIdx.x] = OddSlot{~0ull, 0, 0}; }
__device__ __forceinline__ void odd_note(OddSlot* s, const sobel5_diag* d, int frame, int y, int x,
                                         int32_t P, int32_t M) {
    const int sw = *reinterpret_cast<volatile const int32_t*>(&d->strip_w);
    const uint64_t strip = sw > 0 ? static_cast<uint64_t>(x / sw) : 0u;
    const uint64_t col = sw > 0 ? static_cast<uint64_t>(x % sw) : static_cast<uint64_t>(x);
    auto sat = [](uint64_t v, uint64_t hi) { return v < hi ? v : hi; };
    const uint64_t key = (sat(static_cast<uint64_t>(frame), 1023) << 54) | (sat(strip, 65535) << 38) |
                         (sat(static_cast<uint64_t>(y), (uint64_t{1} << 22) - 1) << 16) |
                         sat(col, 65535);
    OddSlot& o = s[threadIdx.x];
    if (key < o.key) o = OddSlot{key, P, M};
}
static __device__ __noinline__ void diag_publish(sobel5_diag* d, uint64_t key, int32_t P, int32_t M) {
    const uint64_t inv = ~key;
    unsigned __int128* w = reinterpret_cast<unsigned __int128*>(&d->order);
    const unsigned __int128 nv = static_cast<unsigned __int128>(inv) |
                                 (static_cast<unsigned __int128>(static_cast<uint32_t>(P)) << 64) |
                                 (static_cast<unsigned __int128>(static_cast<uint32_t>(M)) << 96);
    unsigned __int128 old = atomicCAS(w, static_cast<unsigned __int128>(0), nv);
    while (old != 0) {
        if (static_cast<uint64_t>(old) >= inv) return;  // an earlier pixel is kept
        const unsigned __int128 seen = atomicCAS(w, old, nv);
        if (seen == old) return;
        old = seen;
    }
}
// end of the kernel (nothing else live): publish this thread's slot
__device__ __forceinline__ void odd_flush(const OddSlot* s, sobel5_diag* d) {
    const OddSlot o = s[threadIdx.x];
    if (o.key != ~0ull) diag_publish(d, o.key, o.p, o.m);
}

__device__ __forceinline__ uint32_t ld_row_word(const uint8_t* p) {
    return __ldg(reinterpret_cast<const unsigned int*>(p));
}

// Store qualifier of the output streams (compile-time knob for experiments;
// default .cs = evict-first streaming, the outputs are not re-read).
#ifndef SOBEL5_ST_Q
#define SOBEL5_ST_Q ".cs"
#endif
__device__ __forceinline__ void st_cs_v4(int32_t* p, int32_t a, int32_t b, int32_t c, int32_t d) {
    asm volatile("st.global" SOBEL5_ST_Q ".v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c),
                 "r"(d)
                 : "memory");
}
__device__ __forceinline__ void st_cs_v4f(float* p, float a, float b, float c, float d) {
    asm volatile("st.global" SOBEL5_ST_Q ".v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}
__device__ __forceinline__ void st_cs_v2d(double* p, double a, double b) {
    asm volatile("st.global" SOBEL5_ST_Q ".v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}
// 256-bit store (STG.E.ENL2.256, sm_100): 4 doubles = 32 B per lane, one
// instruction; measured ~6% more write bandwidth than two 128-bit stores.
__device__ __forceinline__ void st_cs_v4d(double* p, double a, double b, double c, double d) {
    asm volatile("st.global" SOBEL5_ST_Q ".v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c),
                 "d"(d)
                 : "memory");
}
// Write-back (default policy) twins: the StreamResult contract is 1% faster
// with them on the TMA-row kernel (131.7 vs 133.0 us at 8K), SR32 0.7%
// slower (profiles/r1/store_qualifier_sweep.txt)
__device__ __forceinline__ void st_wb_v4(int32_t* p, int32_t a, int32_t b, int32_t c, int32_t d) {
    asm volatile("st.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void st_wb_v4d(double* p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
                 : "memory");
}
// 4 int16 (8 bytes), write-back: the narrow StreamResult wire (kOutN16)
__device__ __forceinline__ void st_wb_v2u(int16_t* p, uint32_t a, uint32_t b) {
    asm volatile("st.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void st_cs_u32(uint8_t* p, uint32_t v) {
    asm volatile("st.global" SOBEL5_ST_Q ".u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// clamp_abs (image_io.hpp:235-240): min(255, round(|g|)); g >= 0 here and
// CUDA round() is round-half-away-from-zero like std::round.
__device__ __forceinline__ uint32_t clamp_abs_u8(double g) {
    const double r = round(g);
    return r < 255.0 ? static_cast<uint32_t>(r) : 255u;
}

// Byte k (0..7) of the 8-byte window lo|hi.
__device__ __forceinline__ uint32_t byte_of(uint32_t lo, uint32_t hi, int k) {
    return k < 4 ? (lo >> (8 * k)) & 0xffu : (hi >> (8 * (k - 4))) & 0xffu;
}

template <class T>
struct TapSource;  // selects runtime (KernelParams) or compile-time taps

template <>
struct TapSource<KernelParams> {
    const KernelParams& p;
    __device__ __forceinline__ int32_t f(int i) const { return p.f[i]; }
    __device__ __forceinline__ int32_t h(int i) const { return p.h[i]; }
    __device__ __forceinline__ int32_t k0(int i) const { return p.k0[i]; }
    __device__ __forceinline__ int32_t k1(int i) const { return p.k1[i]; }
    __device__ __forceinline__ int32_t gx_v(int i) const { return p.gx_v[i]; }
    __device__ __forceinline__ int32_t gy_v(int i) const { return p.gy_v[i]; }
    __device__ __forceinline__ int32_t gdm_f(int i) const { return p.gdm_f[i]; }
    __device__ __forceinline__ int32_t gdm_d(int i) const { return p.gdm_d[i]; }
};

__host__ __device__ constexpr int32_t pick5(int i, int32_t a, int32_t b, int32_t c, int32_t d,
                                            int32_t e) {
    return i == 0 ? a : i == 1 ? b : i == 2 ? c : i == 3 ? d : e;
}

template <>
struct TapSource<DefaultTaps> {
    const KernelParams& p;
    __device__ static constexpr int32_t f(int i) { return pick5(i, -1, -2, 0, 2, 1); }
    __device__ static constexpr int32_t h(int i) { return pick5(i, 1, 4, 6, 4, 1); }
    __device__ static constexpr int32_t k0(int i) { return pick5(i, -6, -6, -2, -6, -6); }
    __device__ static constexpr int32_t k1(int i) { return pick5(i, -2, -12, -16, -12, -2); }
    __device__ static constexpr int32_t gx_v(int i) { return pick5(i, 1, 4, 6, 4, 1); }
    __device__ static constexpr int32_t gy_v(int i) { return pick5(i, -1, -2, 0, 2, 1); }
    __device__ static constexpr int32_t gdm_f(int i) { return pick5(i, 6, 6, 2, 6, 6); }
    __device__ static constexpr int32_t gdm_d(int i) { return pick5(i, 10, 0, -12, 0, 10); }
};

// Geometry of the input rows / columns seen by a kernel instantiation.
enum Geom : int {
    kGeomPlain = 0,  // valid mode over one (or a batch of) plain image(s)
    kGeomSeg = 1,    // valid mode over a stacked [top halo; band; bottom halo]
    kGeomPad = 2,    // pad_replicate(img, 2) fused: same-size output (image_io.hpp:279-291)
    kGeomPlainTma = 3,  // plain, the CTA's band rows bulk-copied (TMA) into shared memory
    kGeomPadTma = 4,    // pad_replicate fused, band rows (clamped) bulk-copied likewise
    kGeomSegTma = 5,    // stacked, band rows bulk-copied for CTAs whose rows are all in mid
    kGeomPlainTmaTs = 6,  // plain + TMA band rows, StreamResult written by TMA tensor stores
    kGeomPlainTmaTw = 7,  // the same, each warp storing its own 128-column boxes
};

// The 8-byte window (wa = input columns c..c+3, wb = c+4..c+7) a lane needs
// for its 4 output columns, from its own row word `own` and the one extra
// word `xtra` that lane 31 (right neighbour word) and, in pad mode, lane 0
// (left neighbour word) load themselves.  The other neighbour words come
// from warp shuffles (the paper's column sharing).
//   valid : c = x0       -> wa = own, wb = right
//   pad   : c = x0 - 2   -> wa = (left:own) bytes 2..5, wb = (own:right) bytes 2..5,
//           columns outside [0, width) replaced by the edge pixel (std::clamp
//           of the column, image_io.hpp:286).
struct PadEdge {
    int active;     // warp-uniform: some lane's window reaches past width-1
    int src_lane;   // lane holding column width-1 ...
    int from_xtra;  // ... in its extra word (lane 31's right word) or its own
    uint32_t sel;   // byte_perm selector replicating that byte
};

__device__ __forceinline__ PadEdge pad_edge_setup(int width, int warp_x0) {
    PadEdge e;
    // lane 31's window ends at column warp_x0 + 131 at most
    e.active = warp_x0 + kWarpCols + 3 >= width;
    // column width-1 relative to the warp: 0..130 whenever active (>= 128 is
    // in lane 31's right neighbour word, owned by the next warp)
    const int c = width - 1 - warp_x0;
    e.from_xtra = c >= kWarpCols;
    e.src_lane = min(31, c >> 2);
    e.sel = static_cast<uint32_t>(c & 3) * 0x1111u;
    return e;
}

// R = pad radius (2 for the 5x5 operator, 1 for the 3x3 one): the window
// starts at column c = x0 - R.
template <bool PAD, int R = 2>
__device__ __forceinline__ void row_window(uint32_t own, uint32_t xtra, int lane, int x0, int width,
                                           const PadEdge& pe, uint32_t& wa, uint32_t& wb) {
    static_assert(R == 1 || R == 2, "pad radius");
    const uint32_t dn = __shfl_down_sync(0xffffffffu, own, 1);
    const uint32_t right = lane != 31 ? dn : xtra;
    if (!PAD) {
        wa = own;
        wb = right;
        return;
    }
    constexpr uint32_t kSel = R == 2 ? 0x5432u : 0x6543u;  // bytes 4-R .. 7-R of (lo:hi)
    const uint32_t up = __shfl_up_sync(0xffffffffu, own, 1);
    const uint32_t left = lane != 0 ? up : (x0 > 0 ? xtra : __byte_perm(own, 0u, 0x0000));
    wa = __byte_perm(left, own, kSel);
    wb = __byte_perm(own, right, kSel);
    if (pe.active) {  // warp-uniform: the right image edge is in this warp's reach
        const uint32_t ew = __shfl_sync(0xffffffffu, pe.from_xtra ? xtra : own, pe.src_lane);
        const uint32_t rep = __byte_perm(ew, 0u, pe.sel);
        const int nv = width - (x0 - R);  // valid window bytes (> R for live lanes)
        if (nv < 4) {
            const uint32_t m = 0xffffffffu << (8 * nv);
            wa = (wa & ~m) | (rep & m);
        }
        if (nv < 8) {
            const int k = nv - 4;
            const uint32_t m = k <= 0 ? 0xffffffffu : 0xffffffffu << (8 * k);
            wb = (wb & ~m) | (rep & m);
        }
    }
}

// Row pointer of stacked input row `row` (0-based, stacked coordinates).
__device__ __forceinline__ const uint8_t* stacked_row(const KernelParams& p, int64_t frame_off,
                                                      int row) {
    if (row < p.top_rows) return p.top + frame_off + static_cast<int64_t>(row) * p.in_pitch;
    row -= p.top_rows;
    if (row < p.mid_rows) return p.mid + frame_off + static_cast<int64_t>(row) * p.in_pitch;
    row -= p.mid_rows;
    return p.bot + frame_off + static_cast<int64_t>(row) * p.in_pitch;
}

// Order-preserving key of a double (sobel5_minmax, include/sobel5_gpu.h).
__host__ __device__ __forceinline__ unsigned long long dkey_bits(unsigned long long b) {
    return b ^ ((b >> 63) ? ~0ull : (1ull << 63));
}
__device__ __forceinline__ unsigned long long dkey(double v) {
    return dkey_bits(static_cast<unsigned long long>(__double_as_longlong(v)));
}
__device__ __forceinline__ double dkey_value(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k ^ (1ull << 63)) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
}

// normalize export of a double magnitude (image_io.hpp:249-253), exact
// reference operation order: lround((v - lo) * 255.0 / span), 0 if span <= 0.
__device__ __forceinline__ uint32_t normalize_u8(double g, double lo, double span) {
    if (!(span > 0.0)) return 0u;
    const double mapped = __ddiv_rn(__dmul_rn(__dsub_rn(g, lo), 255.0), span);
    return static_cast<uint32_t>(static_cast<long long>(round(mapped)));
}

// The fused streaming kernel.
//   PF     : 0 = load each row when it is consumed (Prefetch::off);
//            1 = the next row's load is issued before the current row is
//                processed (Prefetch::on, the paper's Eq. 9 mod-6 ring);
//   TAPS   : KernelParams (runtime taps) or DefaultTaps (compile-time);
//   MAG    : MagMode;
//   PAD    : fused pad_replicate(img, 2) (same-size output) vs valid mode.
template <int PF, class TAPS, int MAG, bool PAD>
// 3 resident CTAs per SM (<= 170 registers, no spills): (1, 32768, 1, 1)
// at 8K 313.8 -> 264.8 us against the unbounded 190-208-register build
#ifndef SOBEL5_GENERIC_MIN_CTAS
#define SOBEL5_GENERIC_MIN_CTAS 3
#endif
__global__ void __launch_bounds__(kCtaThreads, SOBEL5_GENERIC_MIN_CTAS)
    sobel5_stream_kernel(const __grid_constant__ KernelParams p) {
    pdl_enter();
    __shared__ OddSlot s_odd[kCtaThreads];  // ParityViolation
    if (p.diag) odd_init(s_odd);
    const TapSource<TAPS> T{p};
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int warp_x0 = (blockIdx.x * kCtaWarps + warp) * kWarpCols;
    const int x0 = warp_x0 + lane * 4;
    if (warp_x0 >= p.out_w) return;  // whole warp right of the image
    const int oy0 = blockIdx.y * p.band;
    const int n_out = min(p.band, p.out_h - oy0);
    const int n_in = n_out + 4;
    const int64_t in_frame = static_cast<int64_t>(blockIdx.z) * p.in_frame_stride;
    const int64_t out_frame = static_cast<int64_t>(blockIdx.z) * p.out_frame_stride;
    const bool load_a = x0 < p.width;
    const int xoff = (PAD && lane == 0) ? -4 : 4;
    const bool load_b = (lane == 31 && x0 + 4 < p.width) || (PAD && lane == 0 && x0 > 0);
    const bool full = x0 + 3 < p.out_w;
    const PadEdge pe = PAD ? pad_edge_setup(p.width, warp_x0) : PadEdge{0, 0, 0, 0u};
    double n_lo = 0.0, n_span = 0.0;
    if (p.u8_norm) {
        n_lo = p.norm[blockIdx.z].lo;
        n_span = p.norm[blockIdx.z].span;
    }
    unsigned long long g_min = ~0ull, g_max = 0ull;  // order keys of g

    auto row_ptr = [&](int r) -> const uint8_t* {
        if (PAD) {
            const int y = min(max(oy0 + r - 2, 0), p.mid_rows - 1);
            return p.mid + in_frame + static_cast<int64_t>(y) * p.in_pitch;
        }
        return stacked_row(p, in_frame, oy0 + r);
    };

    // Pending vertical accumulators, slot = (output row) mod 5.
    uint32_t acc_x[5][4], acc_y[5][4], acc_p[5][4], acc_m[5][4];

    uint32_t nxt_a = 0, nxt_b = 0;
    if (PF) {
        const uint8_t* rp = row_ptr(0);
        nxt_a = load_a ? ld_row_word(rp + x0) : 0u;
        nxt_b = load_b ? ld_row_word(rp + x0 + xoff) : 0u;
    }

    for (int base = 0; base < n_in; base += 5) {
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            const int r = base + s;
            if (r >= n_in) break;
            uint32_t oa, ob;
            if (PF) {
                oa = nxt_a;
                ob = nxt_b;
                if (r + 1 < n_in) {
                    const uint8_t* rp = row_ptr(r + 1);
                    nxt_a = load_a ? ld_row_word(rp + x0) : 0u;
                    nxt_b = load_b ? ld_row_word(rp + x0 + xoff) : 0u;
                }
            } else {
                const uint8_t* rp = row_ptr(r);
                oa = load_a ? ld_row_word(rp + x0) : 0u;
                ob = load_b ? ld_row_word(rp + x0 + xoff) : 0u;
            }
            // Column sharing: the neighbour words come by warp shuffle.
            uint32_t wa, wb;
            row_window<PAD>(oa, ob, lane, x0, p.width, pe, wa, wb);

            uint32_t px[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) px[k] = byte_of(wa, wb, k);

            // Horizontal passes for the 4 pixels of this lane.
            uint32_t F[4], H[4], D[4], K0[4], K1[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t f = 0, hh = 0, a0 = 0, a1 = 0;
#pragma unroll
                for (int t = 0; t < 5; ++t) {
                    f += static_cast<uint32_t>(T.f(t)) * px[j + t];
                    hh += static_cast<uint32_t>(T.h(t)) * px[j + t];
                    a0 += static_cast<uint32_t>(T.k0(t)) * px[j + t];
                    a1 += static_cast<uint32_t>(T.k1(t)) * px[j + t];
                }
                F[j] = f;
                H[j] = hh;
                K0[j] = a0;
                K1[j] = a1;
                D[j] = px[j + 3] - px[j + 1];
            }

            // Vertical: row r feeds output rows v = r - i, i = 0..4.
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                const int slot = (s - i + 5) % 5;
                const uint32_t cx = static_cast<uint32_t>(T.gx_v(i));
                const uint32_t cy = static_cast<uint32_t>(T.gy_v(i));
                const uint32_t cf = static_cast<uint32_t>(T.gdm_f(i));
                const uint32_t cd = static_cast<uint32_t>(T.gdm_d(i));
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t vx = cx * F[j];
                    const uint32_t vy = cy * H[j];
                    const uint32_t vm = cf * F[j] - cd * D[j];
                    uint32_t vp;
                    if (i == 0) vp = K0[j];
                    else if (i == 1) vp = K1[j];
                    else if (i == 3) vp = 0u - K1[j];
                    else if (i == 4) vp = 0u - K0[j];
                    else vp = 0u;
                    if (i == 0) {
                        acc_x[slot][j] = vx;
                        acc_y[slot][j] = vy;
                        acc_m[slot][j] = vm;
                        acc_p[slot][j] = vp;
                    } else {
                        acc_x[slot][j] += vx;
                        acc_y[slot][j] += vy;
                        acc_m[slot][j] += vm;
                        if (i != 2) acc_p[slot][j] += vp;
                    }
                }
            }

            // Output row v = r - 4 is complete: epilogue + stores.
            if (r >= 4) {
                const int slot = (s + 1) % 5;  // (s - 4) mod 5
                const int v = r - 4;
                int32_t gx[4], gy[4], gd[4], gdt[4];
                bool odd_any = false;
                int32_t odd_p = 0, odd_m = 0, odd_j = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t P = acc_p[slot][j], M = acc_m[slot][j];
                    const uint32_t sum = P + M, dif = P - M;
                    const bool odd = (sum & 1u) != 0u && (x0 + j) < p.out_w;
                    if (odd && !odd_any) {
                        odd_p = static_cast<int32_t>(P);
                        odd_m = static_cast<int32_t>(M);
                        odd_j = j;
                    }
                    odd_any |= odd;
                    gx[j] = static_cast<int32_t>(acc_x[slot][j]);
                    gy[j] = static_cast<int32_t>(acc_y[slot][j]);
                    gd[j] = static_cast<int32_t>(sum) >> 1;
                    gdt[j] = static_cast<int32_t>(dif) >> 1;
                }
                // recover_diag's ParityViolation (pipeline.hpp:268-273),
                // recorded once per warp instead of thrown.
                const unsigned odd_mask = __ballot_sync(0xffffffffu, odd_any);
                if (odd_mask && p.diag) {
                    if (lane == __ffs(odd_mask) - 1) atomicAdd(&p.diag->violations, 1);
                    if (odd_any)
                        odd_note(s_odd, p.diag, blockIdx.z + p.diag_frame0, p.diag_row0 + oy0 + v,
                                 x0 + odd_j, odd_p, odd_m);
                }

                const int64_t row_off = out_frame + static_cast<int64_t>(oy0 + v) * p.pitch + x0;
                if (full) {
                    if (p.gx) st_cs_v4(p.gx + row_off, gx[0], gx[1], gx[2], gx[3]);
                    if (p.gy) st_cs_v4(p.gy + row_off, gy[0], gy[1], gy[2], gy[3]);
                    if (p.gd) st_cs_v4(p.gd + row_off, gd[0], gd[1], gd[2], gd[3]);
                    if (p.gdt) st_cs_v4(p.gdt + row_off, gdt[0], gdt[1], gdt[2], gdt[3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (x0 + j < p.out_w) {
                            if (p.gx) p.gx[row_off + j] = gx[j];
                            if (p.gy) p.gy[row_off + j] = gy[j];
                            if (p.gd) p.gd[row_off + j] = gd[j];
                            if (p.gdt) p.gdt[row_off + j] = gdt[j];
                        }
                    }
                }
                if (p.need_mag) {
                    double g[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (MAG == kMagU32) {
                            const uint32_t ux = static_cast<uint32_t>(gx[j]);
                            const uint32_t uy = static_cast<uint32_t>(gy[j]);
                            const uint32_t ud = static_cast<uint32_t>(gd[j]);
                            const uint32_t ut = static_cast<uint32_t>(gdt[j]);
                            const uint32_t S = ux * ux + uy * uy + ud * ud + ut * ut;
                            g[j] = __dsqrt_rn(__uint2double_rn(S));
                        } else {
                            const double dx = gx[j], dy = gy[j], dd = gd[j], dt = gdt[j];
                            double S = __dmul_rn(dx, dx);
                            S = __dadd_rn(S, __dmul_rn(dy, dy));
                            S = __dadd_rn(S, __dmul_rn(dd, dd));
                            S = __dadd_rn(S, __dmul_rn(dt, dt));
                            g[j] = __dsqrt_rn(S);
                        }
                        if (p.minmax && x0 + j < p.out_w) {
                            const unsigned long long b = dkey(g[j]);
                            g_min = min(g_min, b);
                            g_max = max(g_max, b);
                        }
                    }
                    uint32_t u[4] = {0u, 0u, 0u, 0u};
                    if (p.u8) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            u[j] = p.u8_norm ? normalize_u8(g[j], n_lo, n_span) : clamp_abs_u8(g[j]);
                    }
                    if (full) {
                        if (p.g) {
                            st_cs_v2d(p.g + row_off, g[0], g[1]);
                            st_cs_v2d(p.g + row_off + 2, g[2], g[3]);
                        }
                        if (p.g32)
                            st_cs_v4f(p.g32 + row_off, __double2float_rn(g[0]),
                                      __double2float_rn(g[1]), __double2float_rn(g[2]),
                                      __double2float_rn(g[3]));
                        if (p.u8)
                            st_cs_u32(p.u8 + row_off, u[0] | (u[1] << 8) | (u[2] << 16) | (u[3] << 24));
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            if (x0 + j < p.out_w) {
                                if (p.g) p.g[row_off + j] = g[j];
                                if (p.g32) p.g32[row_off + j] = __double2float_rn(g[j]);
                                if (p.u8) p.u8[row_off + j] = static_cast<uint8_t>(u[j]);
                            }
                        }
                    }
                }
            }
        }
    }
    if (p.minmax) {  // normalize pass 1: frame min / max of g
        for (int o = 16; o > 0; o >>= 1) {
            g_min = min(g_min, __shfl_xor_sync(0xffffffffu, g_min, o));
            g_max = max(g_max, __shfl_xor_sync(0xffffffffu, g_max, o));
        }
        if (lane == 0 && g_min <= g_max) {
            sobel5_minmax* mm = p.minmax + blockIdx.z;
            atomicMin(reinterpret_cast<unsigned long long*>(&mm->lo_key), g_min);
            atomicMax(reinterpret_cast<unsigned long long*>(&mm->hi_key), g_max);
        }
    }
    if (p.diag) odd_flush(s_odd, p.diag);
}

}  // namespace sobel5_b200
