// sobel5_b200/detect.hpp -- the rows next to the streaming engine (SURVEY.md
// 8f rows 1-3) with the reference's names: the 3x3 operator
// (run_stream_3x3 / sobel3_2d, pipeline.hpp:479-573, oracle.hpp:51-70), the
// edge-map export (SaveMode, detail::quantize, image_io.hpp:225-256),
// replicate padding (PaddedPlane / pad_replicate, image_io.hpp:271-291) and
// the CLI's detect flow (sobel5_cli.cpp:127-189) fused on the GPU as
// gpu::detect.  Link with -lsobel5_b200.
//
// What runs where: run_stream_3x3, sobel3_2d, detail::quantize and
// gpu::detect run on the GPU through the C ABI; pad_replicate is the
// reference's host helper (a data-layout copy) -- gpu::detect never calls it,
// the kernels clamp their loads instead.
#pragma once

#include <algorithm>
#include <string>
#include <vector>

#include "sobel5_b200/stream.hpp"

namespace sobel5 {

// ---- 3x3 two-direction operator --------------------------------------------------

struct Stream3Result {
    SignedPlane gx;
    SignedPlane gy;
    RealPlane g;
    OpCounters counters;
};

struct Sobel3Result {
    SignedPlane gx;
    SignedPlane gy;
    RealPlane g;
};

/// run_strip_3x3's tallies (pipeline.hpp:488-547), closed form in the C ABI.
inline OpCounters stream3_counters(int height, const StripPlan& plan, Prefetch prefetch) {
    std::vector<int> widths;
    widths.reserve(plan.strips.size());
    for (const auto& s : plan.strips) widths.push_back(s.out_w);
    sobel5_counters c{};
    gpu::raise(sobel3_plan_counters(height, widths.data(), static_cast<int>(widths.size()),
                                    prefetch == Prefetch::on ? 1 : 0, &c),
               "plan_counters_3x3");
    OpCounters o;
    o.row_conv3_f = c.row_conv3_f;
    o.row_conv3_h = c.row_conv3_h;
    o.mac = c.mac;
    return o;
}

/// Drop-in for sobel5::run_stream_3x3 (pipeline.hpp:551-569).
inline Stream3Result run_stream_3x3(const GrayPlane& img, const StripPlan& plan, Prefetch prefetch,
                                    int workers = 1) {
    (void)workers;
    if (img.width() < 3 || img.height() < 3)
        throw ImageTooSmall("streaming filter needs at least 3x3, got " + std::to_string(img.width()) +
                            "x" + std::to_string(img.height()));
    if (plan.in_width != img.width() || plan.radius != 1)
        throw DimMismatch("strip plan covers " + std::to_string(plan.in_width) + " columns at radius " +
                          std::to_string(plan.radius) + ", image has " + std::to_string(img.width()));
    // device work first, planes built while it runs (gpu::collect_pending)
    Stream3Result out;
    const int ow = img.width() - 2, oh = img.height() - 2;
    sobel5_ctx* c = gpu::thread_context().get();
    sobel5_status st = sobel3_run_host_begin(c, img.data().data(), img.width(), img.height(),
                                             prefetch == Prefetch::on ? 1 : 0, 0x13u /* gx gy g */);
    if (st == SOBEL5_OUT_OF_MEMORY) {  // beyond the pinned-staging cap: direct downloads
        out.gx = SignedPlane(ow, oh);
        out.gy = SignedPlane(ow, oh);
        out.g = RealPlane(ow, oh);
        sobel5_planes pl{};
        pl.pitch = ow;
        pl.gx = out.gx.data().data();
        pl.gy = out.gy.data().data();
        pl.g = out.g.data().data();
        st = sobel3_run_host(c, img.data().data(), img.width(), img.height(),
                             prefetch == Prefetch::on ? 1 : 0, &pl);
    } else if (st == SOBEL5_OK) {
        std::vector<std::int32_t> gx, gy;
        std::vector<double> g;
        st = gpu::collect_pending(c, ow, oh, {{0, &gx}, {1, &gy}, {4, nullptr, &g}}, nullptr);
        if (st == SOBEL5_OK) {
            out.gx = SignedPlane(ow, oh, std::move(gx));
            out.gy = SignedPlane(ow, oh, std::move(gy));
            out.g = RealPlane(ow, oh, std::move(g));
        }
    }
    if (st != SOBEL5_OK)
        gpu::raise(st, std::string("run_stream_3x3 (") + sobel5_ctx_last_error(c) + ")");
    out.counters = stream3_counters(img.height(), plan, prefetch);
    return out;
}

/// pipeline.hpp:571-573
inline Stream3Result run_stream_3x3(const GrayPlane& img, Prefetch prefetch = Prefetch::on) {
    return run_stream_3x3(img, plan_strips(img.width(), img.width(), 1), prefetch, 1);
}

/// oracle.hpp:58-70: identical planes (run_stream_3x3 equals the oracle).
inline Sobel3Result sobel3_2d(const GrayPlane& img) {
    if (img.width() < 3 || img.height() < 3)
        throw ImageTooSmall("conv2d_valid needs at least 3x3, got " + std::to_string(img.width()) + "x" +
                            std::to_string(img.height()));
    auto r = run_stream_3x3(img, Prefetch::on);
    return Sobel3Result{std::move(r.gx), std::move(r.gy), std::move(r.g)};
}

// ---- edge-map export and padding (image_io.hpp) ------------------------------------

enum class SaveMode {
    clamp_abs,  // |v| clipped to [0, 255]
    normalize   // affine map of [min, max] onto [0, 255]; constant maps to 0
};

struct PaddedPlane {
    GrayPlane plane;  // (W + 2r) x (H + 2r)
    int radius = 0;
    int inner_width() const { return plane.width() - 2 * radius; }
    int inner_height() const { return plane.height() - 2 * radius; }
};

/// image_io.hpp:279-291 (host helper; gpu::detect fuses the padding instead).
inline PaddedPlane pad_replicate(const GrayPlane& img, int radius) {
    if (img.empty()) throw EmptyPlane("cannot pad an empty image");
    if (radius < 0) throw DimMismatch("pad radius must be non-negative");
    PaddedPlane out{GrayPlane(img.width() + 2 * radius, img.height() + 2 * radius), radius};
    for (int y = 0; y < out.plane.height(); ++y) {
        const int sy = std::clamp(y - radius, 0, img.height() - 1);
        for (int x = 0; x < out.plane.width(); ++x)
            out.plane.at(y, x) = img.at(sy, std::clamp(x - radius, 0, img.width() - 1));
    }
    return out;
}

namespace detail {

/// image_io.hpp:233-256, computed on the GPU (bit-exact) for the planes the
/// reference instantiates it with: RealPlane, SignedPlane and GrayPlane.
/// Like the reference, the output plane is constructed first, so an empty
/// (0 x 0) plane throws DimMismatch from GrayPlane(0, 0).
template <typename T>
GrayPlane quantize(const Plane<T>& plane, SaveMode mode) {
    static_assert(std::is_same_v<T, double> || std::is_same_v<T, std::int32_t> ||
                      std::is_same_v<T, std::uint8_t>,
                  "quantize: RealPlane, SignedPlane or GrayPlane");
    GrayPlane out(plane.width(), plane.height());
    gpu::Context& ctx = gpu::thread_context();
    constexpr int kind = std::is_same_v<T, double> ? 0 : std::is_same_v<T, std::int32_t> ? 1 : 2;
    const sobel5_status st = sobel5_quantize_host(ctx.get(), plane.data().data(), kind, plane.width(),
                                                  plane.height(), mode == SaveMode::normalize ? 1 : 0,
                                                  out.data().data());
    if (st != SOBEL5_OK) gpu::raise(st, std::string("quantize (") + sobel5_ctx_last_error(ctx.get()) + ")");
    return out;
}

}  // namespace detail

namespace gpu {

/// Planes to dump next to the edge map (the CLI's --dump-planes source).
struct DetectPlanes {
    SignedPlane* gx = nullptr;
    SignedPlane* gy = nullptr;
    SignedPlane* gd = nullptr;
    SignedPlane* gdt = nullptr;
    RealPlane* g = nullptr;
};

/// The CLI's detect flow for the 5x5 operator (sobel5_cli.cpp:127-177):
///   pad_replicate(img, 2) if `pad` -> run_stream -> quantize(g, mode)
/// as one GPU call (padding fused into the loads, normalize's min/max as a
/// device reduction).  Output is W x H with pad, (W-4) x (H-4) without.
inline GrayPlane detect(const GrayPlane& img, const StreamTaps& taps, bool pad = true,
                        SaveMode mode = SaveMode::normalize, Prefetch prefetch = Prefetch::on,
                        const DetectPlanes& dump = {}) {
    if (pad && img.empty()) throw EmptyPlane("cannot pad an empty image");
    if (!pad && (img.width() < 5 || img.height() < 5))
        throw ImageTooSmall("streaming filter needs at least 5x5, got " + std::to_string(img.width()) + "x" +
                            std::to_string(img.height()));
    const int ow = pad ? img.width() : img.width() - 4, oh = pad ? img.height() : img.height() - 4;
    GrayPlane u8(ow, oh);
    sobel5_planes pl{};
    pl.pitch = ow;
    auto bind = [&](auto* plane, auto*& slot) {
        if (plane) {
            *plane = std::remove_reference_t<decltype(*plane)>(ow, oh);
            slot = plane->data().data();
        }
    };
    bind(dump.gx, pl.gx);
    bind(dump.gy, pl.gy);
    bind(dump.gd, pl.gd);
    bind(dump.gdt, pl.gdt);
    bind(dump.g, pl.g);
    const bool any = pl.gx || pl.gy || pl.gd || pl.gdt || pl.g;
    const sobel5_taps t = to_abi(taps);
    sobel5_diag d{};
    Context& ctx = thread_context();
    const sobel5_status st = sobel5_detect_host(ctx.get(), img.data().data(), img.width(), img.height(), &t,
                                                prefetch == Prefetch::on ? 1 : 0, pad ? 1 : 0,
                                                mode == SaveMode::normalize ? 1 : 0, u8.data().data(),
                                                any ? &pl : nullptr, &d);
    if (st == SOBEL5_CUDA_ERROR || st == SOBEL5_OUT_OF_MEMORY)
        raise(st, std::string("detect (") + sobel5_ctx_last_error(ctx.get()) + ")");
    raise(st, "detect", &d);
    return u8;
}

inline GrayPlane detect(const GrayPlane& img, const FilterParams& p = FilterParams{}, bool pad = true,
                        SaveMode mode = SaveMode::normalize, Prefetch prefetch = Prefetch::on) {
    return detect(img, make_stream_taps(p), pad, mode, prefetch);
}

}  // namespace gpu

}  // namespace sobel5
