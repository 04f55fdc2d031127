// cpp_e2e.cpp -- end-to-end timing of the drop-in C++ API on one image
// (default 7680x4320, BASELINE C3), split into its parts:
//   run_stream      sobel5::run_stream as a user calls it (allocates the five
//                   StreamResult planes, host image in, planes out)
//   alloc_planes    just the five value-initialised planes (the reference's
//                   Plane(w, h) zero-fills too, plane.hpp:21)
//   run_host_pageable  sobel5_run_host into already-allocated std::vector planes
//   run_host_pinned    sobel5_run_host into cudaMallocHost planes
//   run_stream_3x3     sobel5::run_stream_3x3 (gx, gy, g: 16 B/px) as a user calls it
// Prints one JSON line.  Build: tools/build_cpp.sh; run on the GPU box.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sobel5_b200/sobel5.hpp"

using namespace sobel5;
using clk = std::chrono::steady_clock;

template <class F>
static double time_ms(int iters, F&& f) {
    f();  // warm-up
    const auto t0 = clk::now();
    for (int i = 0; i < iters; ++i) f();
    return std::chrono::duration<double, std::milli>(clk::now() - t0).count() / iters;
}

int main(int argc, char** argv) {
    const int w = argc > 1 ? std::atoi(argv[1]) : 7680;
    const int h = argc > 2 ? std::atoi(argv[2]) : 4320;
    const int iters = argc > 3 ? std::atoi(argv[3]) : 10;
    const GrayPlane img = synth_random(w, h, 1);
    const StreamTaps taps = make_stream_taps(FilterParams{});
    const StripPlan plan = plan_strips(w, 256, 2);
    const int ow = w - 4, oh = h - 4;
    const double px = double(w) * h;

    StreamResult keep;
    const double t_run = time_ms(iters, [&] { keep = run_stream(img, taps, plan, Prefetch::on); });
    Stream3Result keep3;
    const double t_run3 = time_ms(iters, [&] { keep3 = run_stream_3x3(img, Prefetch::on); });
    const double t_alloc = time_ms(iters, [&] {
        StreamResult r;
        r.gx = SignedPlane(ow, oh);
        r.gy = SignedPlane(ow, oh);
        r.gd = SignedPlane(ow, oh);
        r.gdt = SignedPlane(ow, oh);
        r.g = RealPlane(ow, oh);
    });

    sobel5_ctx* ctx = nullptr;
    if (sobel5_ctx_create(&ctx, 0) != SOBEL5_OK) return 1;
    const sobel5_taps t = gpu::to_abi(taps);
    sobel5_planes pl{};
    pl.pitch = ow;
    pl.gx = keep.gx.data().data();
    pl.gy = keep.gy.data().data();
    pl.gd = keep.gd.data().data();
    pl.gdt = keep.gdt.data().data();
    pl.g = keep.g.data().data();
    sobel5_diag d{};
    const double t_page = time_ms(iters, [&] {
        if (sobel5_run_host(ctx, img.data().data(), w, h, &t, 1, &pl, &d) != SOBEL5_OK) std::exit(2);
    });
    const size_t n = size_t(ow) * oh;
    void* hp[5];
    for (int i = 0; i < 5; ++i)
        if (cudaMallocHost(&hp[i], n * (i == 4 ? 8 : 4)) != cudaSuccess) return 3;
    uint8_t* hin = nullptr;
    if (cudaMallocHost(reinterpret_cast<void**>(&hin), size_t(w) * h) != cudaSuccess) return 3;
    std::memcpy(hin, img.data().data(), size_t(w) * h);
    sobel5_planes pp{};
    pp.pitch = ow;
    pp.gx = static_cast<int32_t*>(hp[0]);
    pp.gy = static_cast<int32_t*>(hp[1]);
    pp.gd = static_cast<int32_t*>(hp[2]);
    pp.gdt = static_cast<int32_t*>(hp[3]);
    pp.g = static_cast<double*>(hp[4]);
    const double t_pin = time_ms(iters, [&] {
        if (sobel5_run_host(ctx, hin, w, h, &t, 1, &pp, &d) != SOBEL5_OK) std::exit(2);
    });
    const bool same = std::memcmp(hp[0], keep.gx.data().data(), n * 4) == 0 &&
                      std::memcmp(hp[4], keep.g.data().data(), n * 8) == 0;
    std::printf(
        "{\"w\": %d, \"h\": %d, \"iters\": %d, \"run_stream_ms\": %.3f, \"run_stream_gpx_s\": %.4f, "
        "\"alloc_planes_ms\": %.3f, \"run_host_pageable_ms\": %.3f, \"run_host_pinned_ms\": %.3f, "
        "\"pinned_gpx_s\": %.4f, \"d2h_bytes\": %zu, \"pinned_equals_pageable\": %s, "
        "\"run_stream_3x3_ms\": %.3f}\n",
        w, h, iters, t_run, px / t_run / 1e6, t_alloc, t_page, t_pin, px / t_pin / 1e6, n * 24,
        same ? "true" : "false", t_run3);
    sobel5_ctx_destroy(ctx);
    return same ? 0 : 4;
}
