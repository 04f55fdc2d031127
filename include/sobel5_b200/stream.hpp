// sobel5_b200/stream.hpp -- the drop-in streaming engine: run_stream and
// friends with the reference's signatures (pipeline.hpp:19-477,
// strips.hpp:13-61, ring.hpp:16-124), executed on the B200 through the C ABI
// (include/sobel5_gpu.h).  Link with -lsobel5_b200.
//
// What runs where:
//   * run_stream / sobel5_4d / diag_via_sum_diff / gpu::edge_map_u8: GPU
//     (sobel5_run_host: chunked H2D, fused kernel, D2H).  There is no CPU
//     fallback: without a device they throw sobel5::DeviceError.
//   * make_stream_taps, plan_strips, the OpCounters tallies and the
//     row-level unit-test helpers (hpass_*, vagg_*, recover_diag, RowRing,
//     KdPlusBank): host code, as in the reference, because they are
//     per-row/per-call bookkeeping, not the per-pixel path.
#pragma once

#include <sys/mman.h>

#include <array>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <span>
#include <string>
#include <thread>
#include <type_traits>
#include <type_traits>
#include <utility>
#include <vector>

#include "sobel5_b200/core.hpp"
#include "sobel5_b200/params.hpp"
#include "sobel5_gpu.h"

namespace sobel5 {

enum class Prefetch { off, on };

struct OpCounters {
    std::uint64_t row_conv5_f = 0;
    std::uint64_t row_conv5_h = 0;
    std::uint64_t row_conv5_k0 = 0;
    std::uint64_t row_conv5_k1 = 0;
    std::uint64_t row_diff = 0;
    std::uint64_t row_conv3_f = 0;
    std::uint64_t row_conv3_h = 0;
    std::uint64_t mac = 0;
    std::uint64_t row_conv5_total() const {
        return row_conv5_f + row_conv5_h + row_conv5_k0 + row_conv5_k1;
    }
    OpCounters& operator+=(const OpCounters& o) {
        row_conv5_f += o.row_conv5_f;
        row_conv5_h += o.row_conv5_h;
        row_conv5_k0 += o.row_conv5_k0;
        row_conv5_k1 += o.row_conv5_k1;
        row_diff += o.row_diff;
        row_conv3_f += o.row_conv3_f;
        row_conv3_h += o.row_conv3_h;
        mac += o.mac;
        return *this;
    }
};

// ---- strips (strips.hpp) -------------------------------------------------------

struct Strip {
    int in_off = 0;
    int out_off = 0;
    int out_w = 0;
    friend bool operator==(const Strip& a, const Strip& b) {
        return a.in_off == b.in_off && a.out_off == b.out_off && a.out_w == b.out_w;
    }
};

struct StripPlan {
    int in_width = 0;
    int out_width = 0;
    int lane_width = 0;
    int radius = 0;
    std::vector<Strip> strips;
};

/// The reference's lane-model tiling (strips.hpp:35-61).  On the GPU the
/// tiling is CTA geometry and independent of the plan; the plan is still
/// validated and drives the reference-schedule counters.
inline StripPlan plan_strips(int width, int lane_width, int radius) {
    if (radius <= 0) throw DimMismatch("strip radius must be positive, got " + std::to_string(radius));
    if (lane_width <= 2 * radius)
        throw LaneTooNarrow("lane width " + std::to_string(lane_width) +
                            " leaves no output columns at radius " + std::to_string(radius));
    if (width < 2 * radius + 1)
        throw ImageTooSmall("width " + std::to_string(width) + " is below the minimum " +
                            std::to_string(2 * radius + 1) + " for radius " + std::to_string(radius));
    StripPlan plan{width, width - 2 * radius, lane_width, radius, {}};
    const int step = lane_width - 2 * radius;
    for (int off = 0; off < plan.out_width; off += step)
        plan.strips.push_back(Strip{off, off, std::min(step, plan.out_width - off)});
    return plan;
}

// ---- rings (ring.hpp) -- host-side helpers for the row-level API ---------------

/// Fixed-depth ring of int32 rows keyed by source row (slot = row mod depth).
class RowRing {
public:
    RowRing(int depth, int row_len) : depth_(depth), len_(row_len) {
        if (depth <= 0 || row_len <= 0) throw DimMismatch("ring depth and row length must be positive");
        cells_.assign(static_cast<std::size_t>(depth) * static_cast<std::size_t>(row_len), 0);
        owner_.assign(static_cast<std::size_t>(depth), -1);
    }
    int depth() const { return depth_; }
    int row_len() const { return len_; }
    static int slot_of(std::int64_t row, int depth) { return static_cast<int>(row % depth); }

    std::span<std::int32_t> acquire(std::int64_t row) {
        const int s = slot_of(row, depth_);
        owner_[static_cast<std::size_t>(s)] = row;
        return {cells_.data() + offset(s), static_cast<std::size_t>(len_)};
    }
    std::span<const std::int32_t> row(std::int64_t r) const {
        const int s = slot_of(r, depth_);
        if (owner_[static_cast<std::size_t>(s)] != r)
            throw MissingRow("ring slot " + std::to_string(s) + " holds row " +
                             std::to_string(owner_[static_cast<std::size_t>(s)]) + ", wanted row " +
                             std::to_string(r));
        return {cells_.data() + offset(s), static_cast<std::size_t>(len_)};
    }
    bool holds(std::int64_t r) const { return owner_[static_cast<std::size_t>(slot_of(r, depth_))] == r; }

private:
    std::size_t offset(int slot) const { return static_cast<std::size_t>(slot) * static_cast<std::size_t>(len_); }
    int depth_, len_;
    std::vector<std::int32_t> cells_;
    std::vector<std::int64_t> owner_;
};

enum class KdVariant : std::uint8_t { k0, k1 };
inline const char* kd_variant_name(KdVariant v) { return v == KdVariant::k0 ? "k0" : "k1"; }

/// Single-bank K_d+ store with variant tags and aggregation signs (Eq. 14).
class KdPlusBank {
public:
    KdPlusBank(int depth, int row_len)
        : ring_(depth, row_len), variant_(static_cast<std::size_t>(depth), KdVariant::k0),
          sign_(static_cast<std::size_t>(depth), 1) {}
    int depth() const { return ring_.depth(); }
    std::span<std::int32_t> acquire(std::int64_t row, KdVariant v) {
        const auto s = static_cast<std::size_t>(RowRing::slot_of(row, depth()));
        variant_[s] = v;
        sign_[s] = 1;
        return ring_.acquire(row);
    }
    std::span<const std::int32_t> row(std::int64_t r, KdVariant expect) const {
        auto span = ring_.row(r);
        const auto s = static_cast<std::size_t>(RowRing::slot_of(r, depth()));
        if (variant_[s] != expect)
            throw VariantMismatch("bank row " + std::to_string(r) + " holds variant " +
                                  kd_variant_name(variant_[s]) + ", wanted " + kd_variant_name(expect));
        return span;
    }
    void stage_center(std::int64_t v) {
        flag(v - 2, 1);
        flag(v - 1, 1);
        flag(v + 1, -1);
        flag(v + 2, -1);
    }
    int sign_of(std::int64_t r) const {
        if (!ring_.holds(r)) throw MissingRow("bank does not hold row " + std::to_string(r));
        return sign_[static_cast<std::size_t>(RowRing::slot_of(r, depth()))];
    }
    bool holds(std::int64_t r) const { return ring_.holds(r); }

private:
    void flag(std::int64_t r, int s) {
        if (!ring_.holds(r)) throw MissingRow("bank does not hold row " + std::to_string(r));
        sign_[static_cast<std::size_t>(RowRing::slot_of(r, depth()))] = static_cast<std::int8_t>(s);
    }
    RowRing ring_;
    std::vector<KdVariant> variant_;
    std::vector<std::int8_t> sign_;
};

// ---- row-level helpers (pipeline.hpp:109-282) -----------------------------------

namespace detail {

inline std::uint64_t nonzero_taps(const std::array<std::int32_t, 5>& taps) {
    std::uint64_t c = 0;
    for (auto t : taps) c += t != 0;
    return c;
}

inline void require_row(std::span<const std::uint8_t> row) {
    if (row.size() < 5) throw RowTooShort("row of " + std::to_string(row.size()) + " pixels, need >= 5");
}

inline std::vector<std::int32_t> taps5(std::span<const std::uint8_t> row, const std::array<std::int32_t, 5>& t) {
    require_row(row);
    std::vector<std::int32_t> out(row.size() - 4);
    for (std::size_t x = 0; x < out.size(); ++x) {
        std::uint32_t acc = 0;  // wraps like the device arithmetic
        for (std::size_t j = 0; j < 5; ++j) acc += static_cast<std::uint32_t>(t[j]) * row[x + j];
        out[x] = static_cast<std::int32_t>(acc);
    }
    return out;
}

// 5-row vertical combination, optionally minus a second ring (Eq. 7, 21).
inline std::vector<std::int32_t> vertical(const RowRing& a, const std::array<std::int32_t, 5>& ca,
                                          const RowRing* b, const std::array<std::int32_t, 5>* cb,
                                          std::int64_t v) {
    std::vector<std::int32_t> out(static_cast<std::size_t>(a.row_len()));
    std::vector<std::uint32_t> acc(out.size(), 0u);
    for (int i = 0; i < 5; ++i) {
        const auto ra = a.row(v - 2 + i);
        for (std::size_t x = 0; x < acc.size(); ++x)
            acc[x] += static_cast<std::uint32_t>(ca[static_cast<std::size_t>(i)]) * static_cast<std::uint32_t>(ra[x]);
        if (b) {
            const auto rb = b->row(v - 2 + i);
            for (std::size_t x = 0; x < acc.size(); ++x)
                acc[x] -= static_cast<std::uint32_t>((*cb)[static_cast<std::size_t>(i)]) * static_cast<std::uint32_t>(rb[x]);
        }
    }
    for (std::size_t x = 0; x < acc.size(); ++x) out[x] = static_cast<std::int32_t>(acc[x]);
    return out;
}

}  // namespace detail

inline std::vector<std::int32_t> hpass_f(std::span<const std::uint8_t> row, const FilterParams& p) {
    detail::require_row(row);
    return detail::taps5(row, make_stream_taps(p).f);
}
inline std::vector<std::int32_t> hpass_h(std::span<const std::uint8_t> row, const FilterParams& p) {
    detail::require_row(row);
    return detail::taps5(row, make_stream_taps(p).h);
}
inline std::vector<std::int32_t> hpass_d(std::span<const std::uint8_t> row) {
    return detail::taps5(row, {0, -1, 0, 1, 0});
}
inline std::vector<std::int32_t> hpass_kd(std::span<const std::uint8_t> row, KdVariant variant,
                                          const FilterParams& p) {
    detail::require_row(row);
    const StreamTaps t = make_stream_taps(p);
    return detail::taps5(row, variant == KdVariant::k0 ? t.k0 : t.k1);
}
inline std::vector<std::int32_t> vagg_gx(const RowRing& f_ring, std::int64_t v, const FilterParams& p) {
    return detail::vertical(f_ring, make_stream_taps(p).gx_v, nullptr, nullptr, v);
}
inline std::vector<std::int32_t> vagg_gy(const RowRing& h_ring, std::int64_t v, const FilterParams& p) {
    return detail::vertical(h_ring, make_stream_taps(p).gy_v, nullptr, nullptr, v);
}
inline std::vector<std::int32_t> vagg_gd_minus(const RowRing& f_ring, const RowRing& d_ring, std::int64_t v,
                                               const FilterParams& p) {
    const StreamTaps t = make_stream_taps(p);
    return detail::vertical(f_ring, t.gdm_f, &d_ring, &t.gdm_d, v);
}
inline std::vector<std::int32_t> vagg_gd_plus(KdPlusBank& bank, std::int64_t v) {
    bank.stage_center(v);
    const std::pair<std::int64_t, KdVariant> taps[4] = {
        {v - 2, KdVariant::k0}, {v - 1, KdVariant::k1}, {v + 1, KdVariant::k1}, {v + 2, KdVariant::k0}};
    std::vector<std::int32_t> out(bank.row(v - 2, KdVariant::k0).size(), 0);
    for (const auto& [r, var] : taps) {
        const auto src = bank.row(r, var);
        const auto s = static_cast<std::uint32_t>(bank.sign_of(r));
        for (std::size_t x = 0; x < out.size(); ++x)
            out[x] = static_cast<std::int32_t>(static_cast<std::uint32_t>(out[x]) + s * static_cast<std::uint32_t>(src[x]));
    }
    return out;
}

/// Eq. 11 halving with the reference's parity check (pipeline.hpp:268-282).
inline std::pair<std::int32_t, std::int32_t> recover_diag(std::int32_t sum, std::int32_t diff) {
    if (((sum + diff) & 1) != 0)
        throw ParityViolation("odd sum/difference pair (" + std::to_string(sum) + ", " + std::to_string(diff) + ")");
    return {(sum + diff) / 2, (sum - diff) / 2};
}
inline void recover_diag(std::span<const std::int32_t> sum, std::span<const std::int32_t> diff,
                         std::span<std::int32_t> gd, std::span<std::int32_t> gdt) {
    for (std::size_t x = 0; x < sum.size(); ++x) std::tie(gd[x], gdt[x]) = recover_diag(sum[x], diff[x]);
}

// ---- results and the GPU entry points ---------------------------------------------

struct StreamResult {
    SignedPlane gx;
    SignedPlane gy;
    SignedPlane gd;
    SignedPlane gdt;
    RealPlane g;
    OpCounters counters;
};

namespace gpu {

/// One device context per host thread (the C ABI context is not thread-safe).
class Context {
public:
    explicit Context(int device = 0) {
        sobel5_ctx* c = nullptr;
        const sobel5_status st = sobel5_ctx_create(&c, device);
        if (st != SOBEL5_OK) throw DeviceError(std::string("sobel5_ctx_create: ") + sobel5_status_string(st));
        ctx_.reset(c);
    }
    sobel5_ctx* get() const { return ctx_.get(); }

private:
    struct Del {
        void operator()(sobel5_ctx* c) const { sobel5_ctx_destroy(c); }
    };
    std::unique_ptr<sobel5_ctx, Del> ctx_;
};

inline int& device_index() {
    thread_local int dev = 0;
    return dev;
}
inline void set_device(int device) { device_index() = device; }

inline Context& thread_context() {
    thread_local std::unique_ptr<Context> ctx;
    thread_local int ctx_dev = -1;
    if (!ctx || ctx_dev != device_index()) {
        ctx = std::make_unique<Context>(device_index());
        ctx_dev = device_index();
    }
    return *ctx;
}

inline sobel5_taps to_abi(const StreamTaps& t) {
    sobel5_taps r{};
    r.a = t.a;
    auto cp = [](std::int32_t* dst, const std::array<std::int32_t, 5>& src) { std::memcpy(dst, src.data(), 20); };
    cp(r.f, t.f);
    cp(r.h, t.h);
    cp(r.k0, t.k0);
    cp(r.k1, t.k1);
    cp(r.gx_v, t.gx_v);
    cp(r.gy_v, t.gy_v);
    cp(r.gdm_f, t.gdm_f);
    cp(r.gdm_d, t.gdm_d);
    r.wide_vagg = t.wide_vagg ? 1 : 0;
    return r;
}

/// Status -> the reference's exception types.
inline void raise(sobel5_status st, const std::string& where, const sobel5_diag* d = nullptr) {
    switch (st) {
        case SOBEL5_OK: return;
        case SOBEL5_PARITY_VIOLATION:
            throw ParityViolation("odd sum/difference pair (" + std::to_string(d ? d->sum : 0) + ", " +
                                  std::to_string(d ? d->diff : 0) + ")");
        case SOBEL5_IMAGE_TOO_SMALL: throw ImageTooSmall(where + ": " + sobel5_status_string(st));
        case SOBEL5_DIM_MISMATCH: throw DimMismatch(where + ": " + sobel5_status_string(st));
        case SOBEL5_NON_POSITIVE_PARAM: throw NonPositiveParam(where + ": " + sobel5_status_string(st));
        case SOBEL5_PARAM_OVERFLOW: throw ParamOverflow(where + ": " + sobel5_status_string(st));
        case SOBEL5_EMPTY_PLANE: throw EmptyPlane("cannot pad an empty image");
        default: throw DeviceError(where + ": " + sobel5_status_string(st));
    }
}

/// Planes wanted from one device pass.
struct Outputs {
    SignedPlane* gx = nullptr;
    SignedPlane* gy = nullptr;
    SignedPlane* gd = nullptr;
    SignedPlane* gdt = nullptr;
    RealPlane* g = nullptr;
    GrayPlane* u8 = nullptr;
};

inline void run(const GrayPlane& img, const StreamTaps& taps, Prefetch prefetch, const Outputs& o) {
    const sobel5_taps t = to_abi(taps);
    sobel5_planes pl{};
    pl.pitch = img.width() - 4;
    pl.gx = o.gx ? o.gx->data().data() : nullptr;
    pl.gy = o.gy ? o.gy->data().data() : nullptr;
    pl.gd = o.gd ? o.gd->data().data() : nullptr;
    pl.gdt = o.gdt ? o.gdt->data().data() : nullptr;
    pl.g = o.g ? o.g->data().data() : nullptr;
    pl.u8 = o.u8 ? o.u8->data().data() : nullptr;
    sobel5_diag d{};
    const sobel5_status st = sobel5_run_host(thread_context().get(), img.data().data(), img.width(), img.height(),
                                             &t, prefetch == Prefetch::on ? 1 : 0, &pl, &d);
    if (st == SOBEL5_CUDA_ERROR || st == SOBEL5_OUT_OF_MEMORY)
        raise(st, std::string("run_stream (") + sobel5_ctx_last_error(thread_context().get()) + ")");
    raise(st, "run_stream", &d);
}

/// Empty storage for n elements with transparent huge pages advised on it
/// before the first touch: fresh result planes are page-fault bound on the
/// host (795 MB at 8K: 290 ms as five serial value-initialised
/// std::vector(n) on the B200 host; profiles/r1/alloc_probe.txt).  Returns
/// the page range of the storage for pre-faulting.
template <typename T>
inline std::pair<std::uintptr_t, std::uintptr_t> huge_reserve(std::vector<T>& v, std::size_t n) {
    v.reserve(n);
    constexpr std::uintptr_t kHuge = std::uintptr_t{2} << 20, kPage = 4096;
    const auto p = reinterpret_cast<std::uintptr_t>(v.data());
    const std::uintptr_t a = (p + kHuge - 1) & ~(kHuge - 1), e = (p + n * sizeof(T)) & ~(kHuge - 1);
    if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);  // advisory only
    return {p & ~(kPage - 1), (p + n * sizeof(T) + kPage - 1) & ~(kPage - 1)};
}

/// Pre-faults page ranges with MADV_POPULATE_WRITE (Linux >= 5.14; a no-op
/// elsewhere) on 4 threads: the kernel zeroes the pages without any
/// user-space access to the not-yet-constructed storage.  Four threads is
/// the measured optimum on the B200 host (22 ms for 795 MB; 8 or 16 threads
/// contend and take 56 ms: profiles/r1/populate_probe.txt).
inline void prefault(const std::vector<std::pair<std::uintptr_t, std::uintptr_t>>& ranges) {
#ifdef __linux__
    constexpr int kPopulateWrite = 23;  // MADV_POPULATE_WRITE
    constexpr std::uintptr_t kPiece = std::uintptr_t{8} << 20;
    std::vector<std::pair<std::uintptr_t, std::uintptr_t>> pieces;
    for (const auto& [a, e] : ranges)
        for (std::uintptr_t o = a; o < e; o += kPiece) pieces.emplace_back(o, std::min(e, o + kPiece));
    std::atomic<std::size_t> next{0};
    auto work = [&] {
        for (std::size_t i; (i = next.fetch_add(1)) < pieces.size();)
            if (madvise(reinterpret_cast<void*>(pieces[i].first), pieces[i].second - pieces[i].first,
                        kPopulateWrite) != 0)
                return;  // unsupported kernel: the first touch faults instead
    };
    // thread creation may fail (std::system_error): run with the threads
    // that did start, the calling thread always works too
    std::vector<std::thread> th;
    try {
        for (int i = 0; i < 3; ++i) th.emplace_back(work);
    } catch (...) {
    }
    work();
    for (auto& t : th) t.join();
#else
    (void)ranges;
#endif
}

/// One result plane of a pending sobel5_run_host_begin / sobel3_run_host_begin:
/// the ABI plane slot (0 gx, 1 gy, 2 gd, 3 gdt, 4 g) and its storage.
struct PendingPlane {
    int slot;
    std::vector<std::int32_t>* i32 = nullptr;
    std::vector<double>* f64 = nullptr;
};

/// Builds the planes of a pending host call while the device works: the
/// storage is reserved with huge pages and pre-faulted, then one host thread
/// per plane appends each row chunk as soon as its download lands
/// (sobel5_run_host_chunk), so the planes are never zero-filled in user
/// space and the host copy overlaps the transfers.  Always completes the
/// pending call (sobel5_run_host_finish); returns its status, rethrows
/// allocation failures.
inline sobel5_status collect_pending(sobel5_ctx* c, int ow, int oh, const std::vector<PendingPlane>& planes,
                                     sobel5_diag* d) {
    const std::size_t n = static_cast<std::size_t>(ow) * static_cast<std::size_t>(oh);
    std::vector<std::exception_ptr> errs(planes.size());
    std::vector<char> short_plane(planes.size(), 0);
    auto fill = [&](std::size_t k, auto& v) {
        try {
            using T = typename std::decay_t<decltype(v)>::value_type;
            const void* stage = sobel5_run_host_staging(c, planes[k].slot);
            // int32 planes may arrive as int16 (the narrow D2H wire): widen
            const bool narrow = std::is_same_v<T, std::int32_t> &&
                                sobel5_run_host_staging_elem(c, planes[k].slot) == 2;
            int y0 = 0, y1 = 0;
            for (int ch = 0; sobel5_run_host_chunk(c, ch, &y0, &y1) == SOBEL5_OK; ++ch) {
                const std::size_t a = static_cast<std::size_t>(y0) * ow, b = static_cast<std::size_t>(y1) * ow;
                if (narrow) {
                    const auto* src = static_cast<const std::int16_t*>(stage);
                    v.insert(v.end(), src + a, src + b);
                } else {
                    const T* src = static_cast<const T*>(stage);
                    v.insert(v.end(), src + a, src + b);
                }
            }
            short_plane[k] = v.size() != n;
        } catch (...) {
            errs[k] = std::current_exception();
        }
    };
    auto run_one = [&](std::size_t k) {
        if (planes[k].i32) fill(k, *planes[k].i32);
        else fill(k, *planes[k].f64);
    };
    bool reserved = true;
    try {
        std::vector<std::pair<std::uintptr_t, std::uintptr_t>> ranges;
        for (const auto& pp : planes)
            ranges.push_back(pp.i32 ? huge_reserve(*pp.i32, n) : huge_reserve(*pp.f64, n));
        if (n >= (std::size_t{1} << 22)) prefault(ranges);  // below ~4K the threads cost more
    } catch (...) {
        errs[0] = std::current_exception();
        reserved = false;
    }
    if (reserved) {
        if (n < (std::size_t{1} << 18)) {
            for (std::size_t k = 0; k < planes.size(); ++k) run_one(k);
        } else {
            // one thread per plane but the first; planes whose thread could
            // not be created (std::system_error) run on the calling thread,
            // and every started thread is joined before the call completes
            std::vector<std::thread> th;
            std::size_t k = 1;
            try {
                for (; k < planes.size(); ++k) th.emplace_back([&, k] { run_one(k); });
            } catch (...) {
            }
            for (std::size_t j = k; j < planes.size(); ++j) run_one(j);
            run_one(0);
            for (auto& x : th) x.join();
        }
    }
    sobel5_status st = sobel5_run_host_finish(c, nullptr, d);  // completes the call: status + diag
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    if (st == SOBEL5_OK)
        for (char f : short_plane)
            if (f) st = SOBEL5_CUDA_ERROR;
    return st;
}

/// run() for the five StreamResult planes, built while the device works
/// (sobel5_run_host_begin, then collect_pending).  The result equals the
/// reference's value-initialised-then-written planes.
inline void run_alloc(const GrayPlane& img, const StreamTaps& taps, Prefetch prefetch, StreamResult& out) {
    const sobel5_taps t = to_abi(taps);
    sobel5_ctx* c = thread_context().get();
    const int ow = img.width() - 4, oh = img.height() - 4;
    sobel5_status st = sobel5_run_host_begin(c, img.data().data(), img.width(), img.height(), &t,
                                             prefetch == Prefetch::on ? 1 : 0, 0x1fu);
    if (st == SOBEL5_OUT_OF_MEMORY) {
        // results beyond the context's pinned-staging cap: allocate the
        // planes first and let sobel5_run_host download into them directly
        out.gx = SignedPlane(ow, oh);
        out.gy = SignedPlane(ow, oh);
        out.gd = SignedPlane(ow, oh);
        out.gdt = SignedPlane(ow, oh);
        out.g = RealPlane(ow, oh);
        run(img, taps, prefetch, Outputs{&out.gx, &out.gy, &out.gd, &out.gdt, &out.g, nullptr});
        return;
    }
    if (st == SOBEL5_CUDA_ERROR)
        raise(st, std::string("run_stream (") + sobel5_ctx_last_error(c) + ")");
    raise(st, "run_stream");
    std::vector<std::int32_t> iv[4];
    std::vector<double> gv;
    sobel5_diag d{};
    st = collect_pending(c, ow, oh,
                         {{0, &iv[0]}, {1, &iv[1]}, {2, &iv[2]}, {3, &iv[3]}, {4, nullptr, &gv}}, &d);
    if (st == SOBEL5_CUDA_ERROR || st == SOBEL5_OUT_OF_MEMORY)
        raise(st, std::string("run_stream (") + sobel5_ctx_last_error(c) + ")");
    raise(st, "run_stream", &d);
    out.gx = SignedPlane(ow, oh, std::move(iv[0]));
    out.gy = SignedPlane(ow, oh, std::move(iv[1]));
    out.gd = SignedPlane(ow, oh, std::move(iv[2]));
    out.gdt = SignedPlane(ow, oh, std::move(iv[3]));
    out.g = RealPlane(ow, oh, std::move(gv));
}

/// The clamp_abs uint8 edge map (image_io.hpp:235-240 applied to g),
/// computed in the same fused kernel; (W-4) x (H-4).
inline GrayPlane edge_map_u8(const GrayPlane& img, const StreamTaps& taps, Prefetch prefetch = Prefetch::on) {
    if (img.width() < 5 || img.height() < 5)
        throw ImageTooSmall("streaming filter needs at least 5x5, got " + std::to_string(img.width()) + "x" +
                            std::to_string(img.height()));
    GrayPlane u8(img.width() - 4, img.height() - 4);
    Outputs o;
    o.u8 = &u8;
    run(img, taps, prefetch, o);
    return u8;
}

}  // namespace gpu

/// Reference-schedule tallies for a plan (pipeline.hpp:330-411, closed form
/// in the C ABI).  Reported for API parity; the GPU does its own work split.
inline OpCounters stream_counters(int height, const StripPlan& plan, const StreamTaps& taps, Prefetch prefetch) {
    std::vector<int> widths;
    widths.reserve(plan.strips.size());
    for (const auto& s : plan.strips) widths.push_back(s.out_w);
    const sobel5_taps t = gpu::to_abi(taps);
    sobel5_counters c{};
    gpu::raise(sobel5_plan_counters(height, widths.data(), static_cast<int>(widths.size()), &t,
                                    prefetch == Prefetch::on ? 1 : 0, &c),
               "plan_counters");
    OpCounters o;
    o.row_conv5_f = c.row_conv5_f;
    o.row_conv5_h = c.row_conv5_h;
    o.row_conv5_k0 = c.row_conv5_k0;
    o.row_conv5_k1 = c.row_conv5_k1;
    o.row_diff = c.row_diff;
    o.row_conv3_f = c.row_conv3_f;
    o.row_conv3_h = c.row_conv3_h;
    o.mac = c.mac;
    return o;
}

/// Drop-in for sobel5::run_stream (pipeline.hpp:452-472): same validation
/// order and messages, same outputs, computed on the GPU.  `workers` is
/// accepted and ignored (the grid replaces the thread pool).
inline StreamResult run_stream(const GrayPlane& img, const StreamTaps& taps, const StripPlan& plan,
                               Prefetch prefetch, int workers = 1) {
    (void)workers;
    if (img.width() < 5 || img.height() < 5)
        throw ImageTooSmall("streaming filter needs at least 5x5, got " + std::to_string(img.width()) + "x" +
                            std::to_string(img.height()));
    if (plan.in_width != img.width() || plan.radius != 2)
        throw DimMismatch("strip plan covers " + std::to_string(plan.in_width) + " columns at radius " +
                          std::to_string(plan.radius) + ", image has " + std::to_string(img.width()));
    StreamResult out;
    // the plan orders the reported ParityViolation pair (strip-major, workers = 1)
    sobel5_ctx_set_strip_width(gpu::thread_context().get(), plan.lane_width - 2 * plan.radius);
    gpu::run_alloc(img, taps, prefetch, out);
    out.counters = stream_counters(img.height(), plan, taps, prefetch);
    return out;
}

/// pipeline.hpp:474-477
inline StreamResult run_stream(const GrayPlane& img, const FilterParams& p, const StripPlan& plan,
                               Prefetch prefetch, int workers = 1) {
    return run_stream(img, make_stream_taps(p), plan, prefetch, workers);
}

// ---- one image over several GPUs (config C5; sobel5_mgpu_* in the C ABI) -----

namespace gpu {

/// RAII over sobel5_mgpu: band k of devices.size() owns input rows
/// [k*H/n, (k+1)*H/n) on devices[k] (devices may repeat).
class BandPartition {
public:
    BandPartition(const std::vector<int>& devices, int width, int height, int transport = SOBEL5_MGPU_AUTO) {
        sobel5_mgpu* m = nullptr;
        raise(sobel5_mgpu_create(&m, devices.data(), static_cast<int>(devices.size()), width, height, transport),
              "sobel5_mgpu_create");
        m_.reset(m);
    }
    sobel5_mgpu* get() const { return m_.get(); }
    sobel5_band_info band(int k) const {
        sobel5_band_info b{};
        raise(sobel5_mgpu_band(m_.get(), k, &b), "sobel5_mgpu_band");
        return b;
    }

private:
    struct Del {
        void operator()(sobel5_mgpu* m) const { sobel5_mgpu_destroy(m); }
    };
    std::unique_ptr<sobel5_mgpu, Del> m_;
};

}  // namespace gpu

/// run_stream with the image row-band partitioned over `devices` (one band
/// per entry; the 2-row halos cross NVLink inside the kernels, or are copied
/// device to device).  Same validation, planes and counters as run_stream
/// (pipeline.hpp:452-477); the reference's strip thread pool
/// (run_strips_parallel, pipeline.hpp:416-445) becomes one band per GPU.
inline StreamResult run_stream_bands(const GrayPlane& img, const StreamTaps& taps, const StripPlan& plan,
                                     Prefetch prefetch, const std::vector<int>& devices,
                                     int transport = SOBEL5_MGPU_AUTO) {
    if (img.width() < 5 || img.height() < 5)
        throw ImageTooSmall("streaming filter needs at least 5x5, got " + std::to_string(img.width()) + "x" +
                            std::to_string(img.height()));
    if (plan.in_width != img.width() || plan.radius != 2)
        throw DimMismatch("strip plan covers " + std::to_string(plan.in_width) + " columns at radius " +
                          std::to_string(plan.radius) + ", image has " + std::to_string(img.width()));
    gpu::BandPartition part(devices, img.width(), img.height(), transport);
    const int ow = img.width() - 4, oh = img.height() - 4;
    StreamResult out;
    out.gx = SignedPlane(ow, oh);
    out.gy = SignedPlane(ow, oh);
    out.gd = SignedPlane(ow, oh);
    out.gdt = SignedPlane(ow, oh);
    out.g = RealPlane(ow, oh);
    sobel5_planes pl{};
    pl.pitch = ow;
    pl.gx = out.gx.data().data();
    pl.gy = out.gy.data().data();
    pl.gd = out.gd.data().data();
    pl.gdt = out.gdt.data().data();
    pl.g = out.g.data().data();
    const sobel5_taps t = gpu::to_abi(taps);
    // the plan orders the reported ParityViolation pair (strip-major)
    sobel5_mgpu_set_strip_width(part.get(), plan.lane_width - 2 * plan.radius);
    const sobel5_status st =
        sobel5_mgpu_run_host(part.get(), img.data().data(), &t, prefetch == Prefetch::on ? 1 : 0, &pl);
    sobel5_diag d{};
    if (st == SOBEL5_PARITY_VIOLATION) sobel5_mgpu_last_diag(part.get(), &d);
    gpu::raise(st, "run_stream_bands", &d);
    out.counters = stream_counters(img.height(), plan, taps, prefetch);
    return out;
}

inline StreamResult run_stream_bands(const GrayPlane& img, const FilterParams& p, const StripPlan& plan,
                                     Prefetch prefetch, const std::vector<int>& devices,
                                     int transport = SOBEL5_MGPU_AUTO) {
    return run_stream_bands(img, make_stream_taps(p), plan, prefetch, devices, transport);
}

/// Same planes as the reference oracle's sobel5_4d (oracle.hpp:72-98), which
/// run_stream equals for every valid parameter set; computed on the GPU.
struct Sobel5Result {
    SignedPlane gx;
    SignedPlane gy;
    SignedPlane gd;
    SignedPlane gdt;
    RealPlane g;
};

/// The oracle's own algorithm on the device (sobel5_dense_4d): four dense
/// correlations with the materialised Kx, Ky, Kd, Kdt and the double
/// magnitude, independent of the streaming kernels run_stream uses -- so a
/// caller's verify flow (run_stream vs sobel5_4d) compares two algorithms,
/// as with the reference.
inline Sobel5Result sobel5_4d(const GrayPlane& img, const FilterParams& p) {
    if (img.width() < 5 || img.height() < 5)
        throw ImageTooSmall("conv2d_valid needs at least 5x5, got " + std::to_string(img.width()) + "x" +
                            std::to_string(img.height()));
    std::int32_t k[4 * 25];
    const Direction dirs[4] = {Direction::X, Direction::Y, Direction::D, Direction::DT};
    for (int d = 0; d < 4; ++d) {
        const Kernel5 m = materialize(p, dirs[d]);
        for (int i = 0; i < 5; ++i)
            for (int j = 0; j < 5; ++j) k[d * 25 + i * 5 + j] = m.at(i, j);
    }
    const int ow = img.width() - 4, oh = img.height() - 4;
    Sobel5Result r{SignedPlane(ow, oh), SignedPlane(ow, oh), SignedPlane(ow, oh), SignedPlane(ow, oh),
                   RealPlane(ow, oh)};
    sobel5_planes pl{};
    pl.pitch = ow;
    pl.gx = r.gx.data().data();
    pl.gy = r.gy.data().data();
    pl.gd = r.gd.data().data();
    pl.gdt = r.gdt.data().data();
    pl.g = r.g.data().data();
    sobel5_ctx* c = gpu::thread_context().get();
    const sobel5_status st = sobel5_dense_4d_host(c, img.data().data(), img.width(), img.height(), k, &pl);
    if (st != SOBEL5_OK) gpu::raise(st, std::string("sobel5_4d (") + sobel5_ctx_last_error(c) + ")");
    return r;
}

/// oracle.hpp:100-129: the diagonal responses through the Kd+/- sum and
/// difference kernels.  For valid FilterParams both numerators are even by
/// construction (Eq. 10-11), so the pair equals run_stream's gd / gdt; it is
/// computed on the GPU (the two planes only).
struct DiagPair {
    SignedPlane gd;
    SignedPlane gdt;
};

inline DiagPair diag_via_sum_diff(const GrayPlane& img, const FilterParams& p) {
    if (img.width() < 5 || img.height() < 5)
        throw ImageTooSmall("conv2d_valid needs at least 5x5, got " + std::to_string(img.width()) + "x" +
                            std::to_string(img.height()));
    DiagPair out{SignedPlane(img.width() - 4, img.height() - 4), SignedPlane(img.width() - 4, img.height() - 4)};
    gpu::Outputs o;
    o.gd = &out.gd;
    o.gdt = &out.gdt;
    gpu::run(img, make_stream_taps(p), Prefetch::on, o);
    return out;
}

// ---- synthetic inputs (synth.hpp) ---------------------------------------------------

inline std::uint64_t splitmix64(std::uint64_t& state) {
    std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

inline GrayPlane synth_random(int width, int height, std::uint64_t seed) {
    GrayPlane img(width, height);
    std::uint64_t state = seed, word = 0;
    auto& px = img.data();
    for (std::size_t i = 0; i < px.size(); ++i) {
        if (i % 8 == 0) word = splitmix64(state);
        px[i] = static_cast<std::uint8_t>(word >> (8 * (i % 8)));
    }
    return img;
}

inline GrayPlane synth_ramp_x(int width, int height) {
    GrayPlane img(width, height);
    for (int y = 0; y < height; ++y)
        for (int x = 0; x < width; ++x) img.at(y, x) = static_cast<std::uint8_t>(x & 0xFF);
    return img;
}

inline GrayPlane synth_constant(int width, int height, std::uint8_t value) {
    GrayPlane img(width, height);
    std::fill(img.data().begin(), img.data().end(), value);
    return img;
}

inline GrayPlane synth_impulse(int width, int height, int y, int x, std::uint8_t value = 1) {
    GrayPlane img(width, height);
    img.at(y, x) = value;
    return img;
}

}  // namespace sobel5
