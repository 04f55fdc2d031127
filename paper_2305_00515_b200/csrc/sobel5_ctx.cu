// sobel5_ctx.cu -- device context and the host-buffer entry point that the
// C++ run_stream wrapper (include/sobel5_b200/sobel5.hpp) calls.
//
// The reference allocates five zero-filled output planes per call
// (pipeline.hpp:462-467) and walks strips on CPU threads (:416-445).  Here a
// context owns the device side once: pitched device planes cached across
// calls, three streams (H2D, compute, D2H) and per-chunk events, so the
// image is processed as row chunks whose upload, kernel and download
// overlap:
//
//   s_h2d : [in 0][in 1][in 2] ...
//   s_comp:       [k 0 ][k 1 ][k 2] ...        (waits on in k)
//   s_d2h :             [out 0    ][out 1 ]... (waits on k k)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "sobel5_gpu.h"

struct sobel5_ctx {
    int device = 0;
    cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
    uint8_t* d_in = nullptr;
    size_t d_in_bytes = 0;
    void* d_plane[7] = {};
    size_t d_plane_bytes[7] = {};
    sobel5_diag* d_diag = nullptr;
    sobel5_diag* h_diag = nullptr;  // pinned
    void* d_scratch = nullptr;      // detect / normalize scratch
    size_t d_scratch_bytes = 0;
    std::vector<cudaEvent_t> ev_in, ev_comp;
    std::string last_error;
};

namespace {

constexpr size_t kElem[7] = {4, 4, 4, 4, 8, 4, 1};  // gx gy gd gdt g g32 u8

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

sobel5_status fail(sobel5_ctx* c, cudaError_t e) {
    c->last_error = cudaGetErrorString(e);
    if (e == cudaErrorMemoryAllocation) return SOBEL5_OUT_OF_MEMORY;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return SOBEL5_NO_DEVICE;
    return SOBEL5_CUDA_ERROR;
}

#define CK(expr)                                        \
    do {                                                \
        cudaError_t e_ = (expr);                        \
        if (e_ != cudaSuccess) return fail(ctx, e_);    \
    } while (0)

cudaError_t ensure(void** p, size_t* cap, size_t bytes) {
    if (*cap >= bytes) return cudaSuccess;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) *cap = bytes;
    return e;
}

cudaError_t ensure_events(std::vector<cudaEvent_t>& v, size_t n) {
    while (v.size() < n) {
        cudaEvent_t ev;
        cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
        v.push_back(ev);
    }
    return cudaSuccess;
}

}  // namespace

extern "C" {

sobel5_status sobel5_ctx_create(sobel5_ctx** out, int device) {
    if (!out) return SOBEL5_INVALID_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return SOBEL5_NO_DEVICE;
    if (device < 0 || device >= n) return SOBEL5_INVALID_ARG;
    auto* ctx = new sobel5_ctx;
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->s_comp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->d_diag, sizeof(sobel5_diag));
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_diag, sizeof(sobel5_diag));
    if (e != cudaSuccess) {
        sobel5_ctx_destroy(ctx);
        return e == cudaErrorMemoryAllocation ? SOBEL5_OUT_OF_MEMORY : SOBEL5_CUDA_ERROR;
    }
    *out = ctx;
    return SOBEL5_OK;
}

void sobel5_ctx_destroy(sobel5_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (auto s : {ctx->s_h2d, ctx->s_comp, ctx->s_d2h})
        if (s) cudaStreamSynchronize(s);
    for (auto ev : ctx->ev_in) cudaEventDestroy(ev);
    for (auto ev : ctx->ev_comp) cudaEventDestroy(ev);
    if (ctx->d_in) cudaFree(ctx->d_in);
    for (void* p : ctx->d_plane)
        if (p) cudaFree(p);
    if (ctx->d_diag) cudaFree(ctx->d_diag);
    if (ctx->d_scratch) cudaFree(ctx->d_scratch);
    if (ctx->h_diag) cudaFreeHost(ctx->h_diag);
    for (auto s : {ctx->s_h2d, ctx->s_comp, ctx->s_d2h})
        if (s) cudaStreamDestroy(s);
    delete ctx;
}

const char* sobel5_ctx_last_error(const sobel5_ctx* ctx) {
    return ctx ? ctx->last_error.c_str() : "";
}

sobel5_status sobel5_run_host(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                              const sobel5_taps* taps, int prefetch, const sobel5_planes* h_out,
                              sobel5_diag* diag_out) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    // pipeline.hpp:454-456 first
    if (width < 5 || height < 5) return SOBEL5_IMAGE_TOO_SMALL;
    if (!h_in || !taps || !h_out) return SOBEL5_INVALID_ARG;
    const int out_w = width - 4, out_h = height - 4;
    if (h_out->pitch != out_w) return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));

    const int64_t in_pitch = round_up(width, 128);
    const int64_t dpitch = round_up(out_w, 32);  // elements; 128 B-aligned int rows
    void* const hp[7] = {h_out->gx, h_out->gy, h_out->gd, h_out->gdt,
                         h_out->g,  h_out->g32, h_out->u8};
    CK(ensure(reinterpret_cast<void**>(&ctx->d_in), &ctx->d_in_bytes,
              static_cast<size_t>(in_pitch) * height));
    sobel5_planes dp{};
    dp.pitch = dpitch;
    void** dslots[7] = {reinterpret_cast<void**>(&dp.gx),  reinterpret_cast<void**>(&dp.gy),
                        reinterpret_cast<void**>(&dp.gd),  reinterpret_cast<void**>(&dp.gdt),
                        reinterpret_cast<void**>(&dp.g),   reinterpret_cast<void**>(&dp.g32),
                        reinterpret_cast<void**>(&dp.u8)};
    for (int i = 0; i < 7; ++i) {
        if (!hp[i]) continue;
        CK(ensure(&ctx->d_plane[i], &ctx->d_plane_bytes[i],
                  static_cast<size_t>(dpitch) * out_h * kElem[i]));
        *dslots[i] = ctx->d_plane[i];
    }

    // Row chunks: enough to overlap copies with compute, few enough that
    // each kernel still fills the GPU.
    int chunk = std::max(256, (out_h + 7) / 8);
    chunk = std::min(chunk, out_h);
    const int n_chunks = (out_h + chunk - 1) / chunk;
    CK(ensure_events(ctx->ev_in, static_cast<size_t>(n_chunks)));
    CK(ensure_events(ctx->ev_comp, static_cast<size_t>(n_chunks)));
    CK(cudaMemsetAsync(ctx->d_diag, 0, sizeof(sobel5_diag), ctx->s_comp));

    int uploaded = 0;  // input rows already enqueued
    for (int k = 0; k < n_chunks; ++k) {
        const int y0 = k * chunk, y1 = std::min(out_h, y0 + chunk);
        const int need = y1 + 4;  // input rows [y0, y1 + 4)
        CK(cudaMemcpy2DAsync(ctx->d_in + static_cast<int64_t>(uploaded) * in_pitch, in_pitch,
                             h_in + static_cast<int64_t>(uploaded) * width, width, width,
                             need - uploaded, cudaMemcpyHostToDevice, ctx->s_h2d));
        uploaded = need;
        CK(cudaEventRecord(ctx->ev_in[k], ctx->s_h2d));
        CK(cudaStreamWaitEvent(ctx->s_comp, ctx->ev_in[k], 0));
        sobel5_planes sub = dp;
        const int64_t off = static_cast<int64_t>(y0) * dpitch;
        if (sub.gx) sub.gx += off;
        if (sub.gy) sub.gy += off;
        if (sub.gd) sub.gd += off;
        if (sub.gdt) sub.gdt += off;
        if (sub.g) sub.g += off;
        if (sub.g32) sub.g32 += off;
        if (sub.u8) sub.u8 += off;
        const sobel5_status st =
            sobel5_launch(ctx->d_in + static_cast<int64_t>(y0) * in_pitch, in_pitch, width,
                          y1 - y0 + 4, taps, prefetch, &sub, ctx->d_diag, ctx->s_comp);
        if (st != SOBEL5_OK) {
            ctx->last_error = cudaGetErrorString(cudaGetLastError());
            return st;
        }
        CK(cudaEventRecord(ctx->ev_comp[k], ctx->s_comp));
        CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_comp[k], 0));
        for (int i = 0; i < 7; ++i) {
            if (!hp[i]) continue;
            const size_t es = kElem[i];
            CK(cudaMemcpy2DAsync(static_cast<char*>(hp[i]) + static_cast<size_t>(y0) * out_w * es,
                                 static_cast<size_t>(out_w) * es,
                                 static_cast<char*>(ctx->d_plane[i]) +
                                     static_cast<size_t>(y0) * dpitch * es,
                                 static_cast<size_t>(dpitch) * es, static_cast<size_t>(out_w) * es,
                                 static_cast<size_t>(y1 - y0), cudaMemcpyDeviceToHost,
                                 ctx->s_d2h));
        }
    }
    CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_comp[n_chunks - 1], 0));
    CK(cudaMemcpyAsync(ctx->h_diag, ctx->d_diag, sizeof(sobel5_diag), cudaMemcpyDeviceToHost,
                       ctx->s_d2h));
    CK(cudaStreamSynchronize(ctx->s_d2h));
    if (diag_out) *diag_out = *ctx->h_diag;
    return ctx->h_diag->violations ? SOBEL5_PARITY_VIOLATION : SOBEL5_OK;
}

sobel5_status sobel5_detect_host(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                                 const sobel5_taps* taps, int prefetch, int pad, int save_mode,
                                 uint8_t* h_u8, const sobel5_planes* h_planes,
                                 sobel5_diag* diag_out) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    if (pad) {
        if (width < 1 || height < 1) return SOBEL5_EMPTY_PLANE;  // image_io.hpp:280
    } else if (width < 5 || height < 5) {
        return SOBEL5_IMAGE_TOO_SMALL;
    }
    if (!h_in || !taps || !h_u8 || (save_mode != 0 && save_mode != 1)) return SOBEL5_INVALID_ARG;
    const int out_w = pad ? width : width - 4, out_h = pad ? height : height - 4;
    if (h_planes && h_planes->pitch != out_w) return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    const int64_t in_pitch = round_up(width, 128);
    const int64_t dpitch = round_up(out_w, 32);
    CK(ensure(reinterpret_cast<void**>(&ctx->d_in), &ctx->d_in_bytes,
              static_cast<size_t>(in_pitch) * height));
    sobel5_planes dp{};
    dp.pitch = dpitch;
    void* hp[7] = {};
    if (h_planes) {
        hp[0] = h_planes->gx; hp[1] = h_planes->gy; hp[2] = h_planes->gd; hp[3] = h_planes->gdt;
        hp[4] = h_planes->g; hp[5] = h_planes->g32;
    }
    hp[6] = h_u8;
    void** dslots[7] = {reinterpret_cast<void**>(&dp.gx),  reinterpret_cast<void**>(&dp.gy),
                        reinterpret_cast<void**>(&dp.gd),  reinterpret_cast<void**>(&dp.gdt),
                        reinterpret_cast<void**>(&dp.g),   reinterpret_cast<void**>(&dp.g32),
                        reinterpret_cast<void**>(&dp.u8)};
    for (int i = 0; i < 7; ++i) {
        if (!hp[i]) continue;
        CK(ensure(&ctx->d_plane[i], &ctx->d_plane_bytes[i],
                  static_cast<size_t>(dpitch) * out_h * kElem[i]));
        *dslots[i] = ctx->d_plane[i];
    }
    CK(ensure(&ctx->d_scratch, &ctx->d_scratch_bytes,
              sobel5_detect_scratch_bytes(out_h, dpitch, 0, 1)));
    CK(cudaMemsetAsync(ctx->d_diag, 0, sizeof(sobel5_diag), ctx->s_comp));
    CK(cudaMemcpy2DAsync(ctx->d_in, in_pitch, h_in, width, width, height, cudaMemcpyHostToDevice,
                         ctx->s_comp));
    const sobel5_status st = sobel5_detect(ctx->d_in, in_pitch, 0, width, height, 1, taps,
                                           prefetch, pad, save_mode, &dp, 0, ctx->d_scratch,
                                           ctx->d_diag, ctx->s_comp);
    if (st != SOBEL5_OK) {
        ctx->last_error = cudaGetErrorString(cudaGetLastError());
        return st;
    }
    for (int i = 0; i < 7; ++i) {
        if (!hp[i]) continue;
        const size_t es = kElem[i];
        CK(cudaMemcpy2DAsync(hp[i], static_cast<size_t>(out_w) * es, ctx->d_plane[i],
                             static_cast<size_t>(dpitch) * es, static_cast<size_t>(out_w) * es,
                             static_cast<size_t>(out_h), cudaMemcpyDeviceToHost, ctx->s_comp));
    }
    CK(cudaMemcpyAsync(ctx->h_diag, ctx->d_diag, sizeof(sobel5_diag), cudaMemcpyDeviceToHost,
                       ctx->s_comp));
    CK(cudaStreamSynchronize(ctx->s_comp));
    if (diag_out) *diag_out = *ctx->h_diag;
    return ctx->h_diag->violations ? SOBEL5_PARITY_VIOLATION : SOBEL5_OK;
}

sobel5_status sobel3_run_host(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                              int prefetch, const sobel5_planes* h_out) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    if (width < 3 || height < 3) return SOBEL5_IMAGE_TOO_SMALL;  // pipeline.hpp:553-556
    if (!h_in || !h_out || h_out->gd || h_out->gdt) return SOBEL5_INVALID_ARG;
    const int out_w = width - 2, out_h = height - 2;
    if (h_out->pitch != out_w) return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    const int64_t in_pitch = round_up(width, 128);
    const int64_t dpitch = round_up(out_w, 32);
    CK(ensure(reinterpret_cast<void**>(&ctx->d_in), &ctx->d_in_bytes,
              static_cast<size_t>(in_pitch) * height));
    sobel5_planes dp{};
    dp.pitch = dpitch;
    void* const hp[7] = {h_out->gx, h_out->gy, nullptr, nullptr, h_out->g, h_out->g32, h_out->u8};
    void** dslots[7] = {reinterpret_cast<void**>(&dp.gx),  reinterpret_cast<void**>(&dp.gy),
                        reinterpret_cast<void**>(&dp.gd),  reinterpret_cast<void**>(&dp.gdt),
                        reinterpret_cast<void**>(&dp.g),   reinterpret_cast<void**>(&dp.g32),
                        reinterpret_cast<void**>(&dp.u8)};
    for (int i = 0; i < 7; ++i) {
        if (!hp[i]) continue;
        CK(ensure(&ctx->d_plane[i], &ctx->d_plane_bytes[i],
                  static_cast<size_t>(dpitch) * out_h * kElem[i]));
        *dslots[i] = ctx->d_plane[i];
    }
    // row chunks: upload / kernel / download overlap as in sobel5_run_host
    int chunk = std::max(256, (out_h + 7) / 8);
    chunk = std::min(chunk, out_h);
    const int n_chunks = (out_h + chunk - 1) / chunk;
    CK(ensure_events(ctx->ev_in, static_cast<size_t>(n_chunks)));
    CK(ensure_events(ctx->ev_comp, static_cast<size_t>(n_chunks)));
    int uploaded = 0;
    for (int k = 0; k < n_chunks; ++k) {
        const int y0 = k * chunk, y1 = std::min(out_h, y0 + chunk);
        const int need = y1 + 2;
        CK(cudaMemcpy2DAsync(ctx->d_in + static_cast<int64_t>(uploaded) * in_pitch, in_pitch,
                             h_in + static_cast<int64_t>(uploaded) * width, width, width,
                             need - uploaded, cudaMemcpyHostToDevice, ctx->s_h2d));
        uploaded = need;
        CK(cudaEventRecord(ctx->ev_in[k], ctx->s_h2d));
        CK(cudaStreamWaitEvent(ctx->s_comp, ctx->ev_in[k], 0));
        sobel5_planes sub = dp;
        const int64_t off = static_cast<int64_t>(y0) * dpitch;
        if (sub.gx) sub.gx += off;
        if (sub.gy) sub.gy += off;
        if (sub.g) sub.g += off;
        if (sub.g32) sub.g32 += off;
        if (sub.u8) sub.u8 += off;
        const sobel5_status st =
            sobel3_launch(ctx->d_in + static_cast<int64_t>(y0) * in_pitch, in_pitch, 0, width,
                          y1 - y0 + 2, 1, prefetch, 0, &sub, 0, ctx->s_comp);
        if (st != SOBEL5_OK) {
            ctx->last_error = cudaGetErrorString(cudaGetLastError());
            return st;
        }
        CK(cudaEventRecord(ctx->ev_comp[k], ctx->s_comp));
        CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_comp[k], 0));
        for (int i = 0; i < 7; ++i) {
            if (!hp[i]) continue;
            const size_t es = kElem[i];
            CK(cudaMemcpy2DAsync(static_cast<char*>(hp[i]) + static_cast<size_t>(y0) * out_w * es,
                                 static_cast<size_t>(out_w) * es,
                                 static_cast<char*>(ctx->d_plane[i]) +
                                     static_cast<size_t>(y0) * dpitch * es,
                                 static_cast<size_t>(dpitch) * es, static_cast<size_t>(out_w) * es,
                                 static_cast<size_t>(y1 - y0), cudaMemcpyDeviceToHost,
                                 ctx->s_d2h));
        }
    }
    CK(cudaStreamSynchronize(ctx->s_d2h));
    return SOBEL5_OK;
}

sobel5_status sobel5_quantize_host(sobel5_ctx* ctx, const void* h_plane, int kind, int width,
                                   int height, int save_mode, uint8_t* h_u8) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    if (width < 1 || height < 1) return SOBEL5_EMPTY_PLANE;  // image_io.hpp:259/265
    if (!h_plane || !h_u8 || (kind != 0 && kind != 1)) return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    const size_t es = kind == 0 ? sizeof(double) : sizeof(int32_t);
    const size_t n = static_cast<size_t>(width) * height;
    // the plane goes through the g slot (8 B/elem covers both kinds), u8 through u8
    CK(ensure(&ctx->d_plane[4], &ctx->d_plane_bytes[4], n * 8));
    CK(ensure(&ctx->d_plane[6], &ctx->d_plane_bytes[6], n));
    CK(ensure(&ctx->d_scratch, &ctx->d_scratch_bytes, sobel5_detect_scratch_bytes(0, 0, 0, 1)));
    CK(cudaMemcpyAsync(ctx->d_plane[4], h_plane, n * es, cudaMemcpyHostToDevice, ctx->s_comp));
    const sobel5_status st =
        sobel5_quantize_plane(ctx->d_plane[4], kind, width, width, height, save_mode,
                              static_cast<uint8_t*>(ctx->d_plane[6]), width, ctx->d_scratch,
                              ctx->s_comp);
    if (st != SOBEL5_OK) return st;
    CK(cudaMemcpyAsync(h_u8, ctx->d_plane[6], n, cudaMemcpyDeviceToHost, ctx->s_comp));
    CK(cudaStreamSynchronize(ctx->s_comp));
    return SOBEL5_OK;
}

}  // extern "C"
