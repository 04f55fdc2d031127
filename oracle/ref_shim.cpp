// ref_shim.cpp -- extern "C" face over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE (see oracle/sobel5_oracle.h).  Compiled by
// oracle/Makefile directly against /root/reference/proj/include (the
// reference's own sources, never copied into this repo) into
// oracle/_ref/libsobel5_ref.so.  Used by tests/ to pin the C restatement and
// to make golden fixtures, and by bench.py --impl reference / cpu_baseline as
// the reference's own CPU implementation of the path.
//
// image_io.hpp #includes <png.h>; libpng is absent here, so the Makefile puts
// a declaration-only stand-in (oracle/png_stub/png.h) on the include path.
// Only its pure-C++ pieces are called (detail::quantize, pad_replicate);
// the shim links with -Wl,--no-undefined, proving no libpng symbol is used.
#include <cstring>
#include <exception>
#include <string>

#include "sobel5/filter_algebra.hpp"
#include "sobel5/image_io.hpp"
#include "sobel5/metrics.hpp"
#include "sobel5/oracle.hpp"
#include "sobel5/pipeline.hpp"
#include "sobel5/strips.hpp"
#include "sobel5/synth.hpp"

namespace {

struct RefTaps {  // same layout as oracle_taps / sobel5_taps
    std::int32_t a;
    std::int32_t f[5], h[5], k0[5], k1[5], gx_v[5], gy_v[5], gdm_f[5], gdm_d[5];
    std::int32_t wide_vagg;
};

sobel5::StreamTaps to_taps(const RefTaps& r) {
    sobel5::StreamTaps t;
    t.a = r.a;
    for (int i = 0; i < 5; ++i) {
        t.f[i] = r.f[i];
        t.h[i] = r.h[i];
        t.k0[i] = r.k0[i];
        t.k1[i] = r.k1[i];
        t.gx_v[i] = r.gx_v[i];
        t.gy_v[i] = r.gy_v[i];
        t.gdm_f[i] = r.gdm_f[i];
        t.gdm_d[i] = r.gdm_d[i];
    }
    t.wide_vagg = r.wide_vagg != 0;
    return t;
}

void from_taps(const sobel5::StreamTaps& t, RefTaps* r) {
    r->a = t.a;
    for (int i = 0; i < 5; ++i) {
        r->f[i] = t.f[i];
        r->h[i] = t.h[i];
        r->k0[i] = t.k0[i];
        r->k1[i] = t.k1[i];
        r->gx_v[i] = t.gx_v[i];
        r->gy_v[i] = t.gy_v[i];
        r->gdm_f[i] = t.gdm_f[i];
        r->gdm_d[i] = t.gdm_d[i];
    }
    r->wide_vagg = t.wide_vagg ? 1 : 0;
}

// Error classes -> small integers, in errors.hpp declaration order.
int classify(const std::exception& e) {
    using namespace sobel5;
    if (dynamic_cast<const NonPositiveParam*>(&e)) return 10;
    if (dynamic_cast<const NonIntegralWeight*>(&e)) return 11;
    if (dynamic_cast<const ParamOverflow*>(&e)) return 12;
    if (dynamic_cast<const ImageTooSmall*>(&e)) return 13;
    if (dynamic_cast<const RowTooShort*>(&e)) return 14;
    if (dynamic_cast<const MissingRow*>(&e)) return 15;
    if (dynamic_cast<const VariantMismatch*>(&e)) return 16;
    if (dynamic_cast<const ParityViolation*>(&e)) return 17;
    if (dynamic_cast<const LaneTooNarrow*>(&e)) return 18;
    if (dynamic_cast<const DimMismatch*>(&e)) return 19;
    if (dynamic_cast<const EmptyPlane*>(&e)) return 20;
    return 99;
}

int report(const std::exception& e, char* err, int errlen) {
    if (err && errlen > 0) {
        std::strncpy(err, e.what(), static_cast<std::size_t>(errlen) - 1);
        err[errlen - 1] = 0;
    }
    return classify(e);
}

sobel5::Rational rat(std::int64_t num, std::int64_t den) { return sobel5::Rational(num, den); }

void copy_plane(const sobel5::SignedPlane& p, std::int32_t* dst) {
    if (dst) std::memcpy(dst, p.data().data(), p.size() * sizeof(std::int32_t));
}

}  // namespace

extern "C" {

int ref_make_stream_taps(std::int64_t a, std::int64_t bn, std::int64_t bd, std::int64_t mn,
                         std::int64_t md, std::int64_t nn, std::int64_t nd, RefTaps* out,
                         char* err, int errlen) {
    try {
        sobel5::FilterParams p;
        p.a = a;
        p.b = rat(bn, bd);
        p.m = rat(mn, md);
        p.n = rat(nn, nd);
        from_taps(sobel5::make_stream_taps(p), out);
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

int ref_materialize(std::int64_t a, std::int64_t b, std::int64_t m, std::int64_t n, int dir,
                    std::int32_t* k25, char* err, int errlen) {
    try {
        sobel5::FilterParams p;
        p.a = a;
        p.b = b;
        p.m = m;
        p.n = n;
        sobel5::validate_params(p);
        const auto k = sobel5::materialize(p, static_cast<sobel5::Direction>(dir));
        for (int i = 0; i < 5; ++i)
            for (int j = 0; j < 5; ++j) k25[i * 5 + j] = k.w[i][j];
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

int ref_run_stream(const std::uint8_t* img, int w, int h, const RefTaps* taps, int lanes,
                   int prefetch, int workers, std::int32_t* gx, std::int32_t* gy,
                   std::int32_t* gd, std::int32_t* gdt, double* g, std::uint64_t* counters8,
                   char* err, int errlen) {
    try {
        sobel5::GrayPlane in(w, h, std::vector<std::uint8_t>(img, img + std::size_t(w) * h));
        const auto plan = sobel5::plan_strips(w, lanes, 2);
        const auto r = sobel5::run_stream(in, to_taps(*taps), plan,
                                          prefetch ? sobel5::Prefetch::on : sobel5::Prefetch::off,
                                          workers);
        copy_plane(r.gx, gx);
        copy_plane(r.gy, gy);
        copy_plane(r.gd, gd);
        copy_plane(r.gdt, gdt);
        if (g) std::memcpy(g, r.g.data().data(), r.g.size() * sizeof(double));
        if (counters8) {
            const auto& c = r.counters;
            const std::uint64_t v[8] = {c.row_conv5_f, c.row_conv5_h, c.row_conv5_k0,
                                        c.row_conv5_k1, c.row_diff,   c.row_conv3_f,
                                        c.row_conv3_h, c.mac};
            std::memcpy(counters8, v, sizeof v);
        }
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

int ref_sobel5_4d(const std::uint8_t* img, int w, int h, std::int64_t a, std::int64_t b,
                  std::int64_t m, std::int64_t n, std::int32_t* gx, std::int32_t* gy,
                  std::int32_t* gd, std::int32_t* gdt, double* g, char* err, int errlen) {
    try {
        sobel5::GrayPlane in(w, h, std::vector<std::uint8_t>(img, img + std::size_t(w) * h));
        sobel5::FilterParams p;
        p.a = a;
        p.b = b;
        p.m = m;
        p.n = n;
        const auto r = sobel5::sobel5_4d(in, p);
        copy_plane(r.gx, gx);
        copy_plane(r.gy, gy);
        copy_plane(r.gd, gd);
        copy_plane(r.gdt, gdt);
        if (g) std::memcpy(g, r.g.data().data(), r.g.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

int ref_diag_via_sum_diff(const std::uint8_t* img, int w, int h, std::int32_t* gd,
                          std::int32_t* gdt, char* err, int errlen) {
    try {
        sobel5::GrayPlane in(w, h, std::vector<std::uint8_t>(img, img + std::size_t(w) * h));
        const auto r = sobel5::diag_via_sum_diff(in, sobel5::FilterParams{});
        copy_plane(r.gd, gd);
        copy_plane(r.gdt, gdt);
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

void ref_synth_random(std::uint8_t* img, int w, int h, std::uint64_t seed) {
    const auto p = sobel5::synth_random(w, h, seed);
    std::memcpy(img, p.data().data(), p.size());
}

int ref_plan_strips(int width, int lanes, int radius, int max_strips, int* n_strips, int* in_off,
                    int* out_off, int* out_w, char* err, int errlen) {
    try {
        const auto plan = sobel5::plan_strips(width, lanes, radius);
        *n_strips = static_cast<int>(plan.strips.size());
        for (int i = 0; i < *n_strips && i < max_strips; ++i) {
            in_off[i] = plan.strips[static_cast<std::size_t>(i)].in_off;
            out_off[i] = plan.strips[static_cast<std::size_t>(i)].out_off;
            out_w[i] = plan.strips[static_cast<std::size_t>(i)].out_w;
        }
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

// Row-level public helpers (pipeline.hpp:194-233, 268-273): which = 0 f,
// 1 h, 2 d, 3 kd k0, 4 kd k1.
int ref_hpass(const std::uint8_t* row, int len, int which, std::int64_t a, std::int64_t b,
              std::int64_t m, std::int64_t n, std::int32_t* out, char* err, int errlen) {
    try {
        sobel5::FilterParams p;
        p.a = a;
        p.b = b;
        p.m = m;
        p.n = n;
        std::span<const std::uint8_t> r(row, static_cast<std::size_t>(len));
        std::vector<std::int32_t> v;
        switch (which) {
            case 0: v = sobel5::hpass_f(r, p); break;
            case 1: v = sobel5::hpass_h(r, p); break;
            case 2: v = sobel5::hpass_d(r); break;
            case 3: v = sobel5::hpass_kd(r, sobel5::KdVariant::k0, p); break;
            default: v = sobel5::hpass_kd(r, sobel5::KdVariant::k1, p); break;
        }
        std::memcpy(out, v.data(), v.size() * sizeof(std::int32_t));
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

int ref_recover_diag(std::int32_t sum, std::int32_t diff, std::int32_t* gd, std::int32_t* gdt,
                     char* err, int errlen) {
    try {
        const auto [d, t] = sobel5::recover_diag(sum, diff);
        *gd = d;
        *gdt = t;
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

// The reference's own timing harness (metrics.hpp:142-179) around its own
// run_stream (pipeline.hpp:474): 1 untimed warm-up + `iters` timed calls.
// Returns mean seconds per call; stddev via *stddev_s.
double ref_measure_run_stream(const std::uint8_t* img, int w, int h, int lanes, int prefetch,
                              int workers, int iters, double* stddev_s) {
    sobel5::GrayPlane in(w, h, std::vector<std::uint8_t>(img, img + std::size_t(w) * h));
    const auto plan = sobel5::plan_strips(w, lanes, 2);
    const sobel5::FilterParams p;
    const auto rep = sobel5::measure("fast-5x5", w, h, iters, workers, [&] {
        auto r = sobel5::run_stream(in, p, plan,
                                    prefetch ? sobel5::Prefetch::on : sobel5::Prefetch::off,
                                    workers);
        (void)r;
    });
    if (stddev_s) *stddev_s = rep.stddev_s;
    return rep.mean_s;
}

// The reference CLI's bench rows (sobel5_cli.cpp:236-276): measure() of
// run_stream ("fast-5x5", which = 0) or of the sobel5_4d oracle
// ("oracle-5x5", which = 1, one worker).  out[0..3] = the BenchReport's
// mean_s, stddev_s, mps, mps_per_core (pyoracle formats the reference's CSV
// row, metrics.hpp:129-139, from them).  Returns mean_s.
double ref_measure_csv(const std::uint8_t* img, int w, int h, int which, int lanes, int prefetch,
                       int workers, int iters, double* out) {
    sobel5::GrayPlane in(w, h, std::vector<std::uint8_t>(img, img + std::size_t(w) * h));
    const sobel5::FilterParams p;
    sobel5::BenchReport rep;
    if (which == 0) {
        const auto plan = sobel5::plan_strips(w, lanes, 2);
        rep = sobel5::measure("fast-5x5", w, h, iters, workers, [&] {
            auto r = sobel5::run_stream(in, p, plan,
                                        prefetch ? sobel5::Prefetch::on : sobel5::Prefetch::off,
                                        workers);
            (void)r;
        });
    } else {
        rep = sobel5::measure("oracle-5x5", w, h, iters, 1, [&] {
            auto r = sobel5::sobel5_4d(in, p);
            (void)r;
        });
    }
    out[0] = rep.mean_s;
    out[1] = rep.stddev_s;
    out[2] = rep.mps;
    out[3] = rep.mps_per_core;
    return rep.mean_s;
}

double ref_measure_oracle(const std::uint8_t* img, int w, int h, int iters) {
    sobel5::GrayPlane in(w, h, std::vector<std::uint8_t>(img, img + std::size_t(w) * h));
    const auto rep = sobel5::measure("oracle-5x5", w, h, iters, 1, [&] {
        auto r = sobel5::sobel5_4d(in, sobel5::FilterParams{});
        (void)r;
    });
    return rep.mean_s;
}

// ---- detect path pieces -------------------------

// pad_replicate (image_io.hpp:279-291); out is (w+2r) x (h+2r).
int ref_pad_replicate(const std::uint8_t* img, int w, int h, int r, std::uint8_t* out, char* err,
                      int errlen) {
    try {
        sobel5::GrayPlane in = w > 0 && h > 0
            ? sobel5::GrayPlane(w, h, std::vector<std::uint8_t>(img, img + std::size_t(w) * h))
            : sobel5::GrayPlane();
        const auto p = sobel5::pad_replicate(in, r);
        std::memcpy(out, p.plane.data().data(), p.plane.size());
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

// detail::quantize (image_io.hpp:233-256) of a RealPlane (kind 0) or a
// SignedPlane (kind 1); mode 0 = clamp_abs, 1 = normalize.
int ref_quantize(const void* plane, int kind, int w, int h, int mode, std::uint8_t* out) {
    const auto m = mode ? sobel5::SaveMode::normalize : sobel5::SaveMode::clamp_abs;
    const std::size_t n = std::size_t(w) * h;
    sobel5::GrayPlane q;
    if (kind == 0) {
        const double* v = static_cast<const double*>(plane);
        q = sobel5::detail::quantize(sobel5::RealPlane(w, h, std::vector<double>(v, v + n)), m);
    } else {
        const std::int32_t* v = static_cast<const std::int32_t*>(plane);
        q = sobel5::detail::quantize(
            sobel5::SignedPlane(w, h, std::vector<std::int32_t>(v, v + n)), m);
    }
    std::memcpy(out, q.data().data(), q.size());
    return 0;
}

// sobel3_2d (oracle.hpp:58-70).
int ref_sobel3_2d(const std::uint8_t* img, int w, int h, std::int32_t* gx, std::int32_t* gy,
                  double* g, char* err, int errlen) {
    try {
        sobel5::GrayPlane in(w, h, std::vector<std::uint8_t>(img, img + std::size_t(w) * h));
        const auto r = sobel5::sobel3_2d(in);
        copy_plane(r.gx, gx);
        copy_plane(r.gy, gy);
        if (g) std::memcpy(g, r.g.data().data(), r.g.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

// run_stream_3x3 (pipeline.hpp:551-573) with plan_strips(w, lanes, 1).
int ref_run_stream_3x3(const std::uint8_t* img, int w, int h, int lanes, int prefetch,
                       int workers, std::int32_t* gx, std::int32_t* gy, double* g,
                       std::uint64_t* counters8, char* err, int errlen) {
    try {
        sobel5::GrayPlane in(w, h, std::vector<std::uint8_t>(img, img + std::size_t(w) * h));
        const auto plan = sobel5::plan_strips(w, lanes, 1);
        const auto r = sobel5::run_stream_3x3(
            in, plan, prefetch ? sobel5::Prefetch::on : sobel5::Prefetch::off, workers);
        copy_plane(r.gx, gx);
        copy_plane(r.gy, gy);
        if (g) std::memcpy(g, r.g.data().data(), r.g.size() * sizeof(double));
        if (counters8) {
            const auto& c = r.counters;
            const std::uint64_t v[8] = {c.row_conv5_f, c.row_conv5_h, c.row_conv5_k0,
                                        c.row_conv5_k1, c.row_diff,   c.row_conv3_f,
                                        c.row_conv3_h, c.mac};
            std::memcpy(counters8, v, sizeof v);
        }
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

// The reference's timing harness around its run_stream_3x3.
double ref_measure_run_stream_3x3(const std::uint8_t* img, int w, int h, int lanes, int prefetch,
                                  int workers, int iters, double* stddev_s) {
    sobel5::GrayPlane in(w, h, std::vector<std::uint8_t>(img, img + std::size_t(w) * h));
    const auto plan = sobel5::plan_strips(w, lanes, 1);
    const auto rep = sobel5::measure("fast-3x3", w, h, iters, workers, [&] {
        auto r = sobel5::run_stream_3x3(
            in, plan, prefetch ? sobel5::Prefetch::on : sobel5::Prefetch::off, workers);
        (void)r;
    });
    if (stddev_s) *stddev_s = rep.stddev_s;
    return rep.mean_s;
}

// conv2d_valid (oracle.hpp:19-49) with an arbitrary 5x5 / 3x3 kernel.
int ref_conv2d_valid(const std::uint8_t* img, int w, int h, const std::int32_t* k, int ksize,
                     std::int32_t* out) {
    try {
        const sobel5::GrayPlane g(w, h, std::vector<std::uint8_t>(img, img + std::size_t(w) * h));
        sobel5::SignedPlane r;
        if (ksize == 5) {
            sobel5::Kernel5 kk;
            for (int i = 0; i < 5; ++i)
                for (int j = 0; j < 5; ++j) kk.w[i][j] = k[i * 5 + j];
            r = sobel5::conv2d_valid(g, kk);
        } else {
            sobel5::Kernel3 kk;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) kk.w[i][j] = k[i * 3 + j];
            r = sobel5::conv2d_valid(g, kk);
        }
        copy_plane(r, out);
        return 0;
    } catch (const std::exception& e) {
        return classify(e);
    }
}

}  // extern "C"
