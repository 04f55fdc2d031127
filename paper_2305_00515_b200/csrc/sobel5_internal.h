// sobel5_internal.h -- library-internal launch interface shared by the
// translation units (kernels are instantiated in separate .cu files so the
// build compiles them in parallel).  Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <utility>

#include <cstdint>

#include "sobel5_gpu.h"
#include "sobel5_stream.cuh"

namespace sobel5_b200 {

// PDL on the stream kernels (SOBEL5_PDL, default 1; see pdl_enter()).
bool pdl_enabled();

// Launches kernel k(kp) with the programmatic-stream-serialization
// attribute when PDL is enabled (every kernel launched this way calls
// pdl_enter() first).
template <typename Kernel>
cudaError_t launch_kp(Kernel k, dim3 grid, int threads, size_t smem, cudaStream_t s,
                      const KernelParams& kp) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, kp);
}

// The same for any kernel signature (the detect path's small kernels).
template <typename... P, typename... A>
cudaError_t launch_pdl(void (*k)(P...), dim3 grid, dim3 block, cudaStream_t s, A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

// Packed default-taps kernel (sobel5_packed.cuh), one launcher per geometry.
cudaError_t launch_packed_plain(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s);
cudaError_t launch_packed_seg(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s);
cudaError_t launch_packed_pad(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s);

// Packed kernel with runtime taps (any taps within the int16 bound).
cudaError_t launch_packed_rt_plain(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s);
cudaError_t launch_packed_rt_seg(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s);
cudaError_t launch_packed_rt_pad(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s);

// u8-only clamp_abs contract, default taps (sobel5_u8.cuh): 2NP px per lane,
// TMA band rows; its own grid (W warps x 32 x 2NP columns per CTA) and band.
struct U8Plan {
    int np = 4, warps = 4, band = 16, cta_cols = 1024;
};
U8Plan u8_fast_plan(int out_w, int out_h, int frames);
cudaError_t launch_u8_fast(const KernelParams& kp, int frames, const U8Plan& plan, cudaStream_t s);
// The same for the 3x3 operator's u8-only contract (sobel3_u8.cuh).
U8Plan u3_fast_plan(int out_w, int out_h, int frames);
cudaError_t launch_u3_fast(const KernelParams& kp, int frames, const U8Plan& plan, cudaStream_t s);

// Tensor maps of the StreamResult planes for the TMA-store kernel
// (sobel5_tmap.cu); false if the driver entry point or the layout is missing.
bool build_store_maps(KernelParams& kp, int frames, int rows, int box_cols);

// Packed-FP32 kernel with runtime taps (sobel5_f32x2.cuh), every geometry.
cudaError_t launch_f32(const KernelParams& kp, dim3 grid, int pf, MagMode mag, cudaStream_t s);

// Ablation only: default taps as four dense 5x5 correlations (sobel5_k_dense.cu).
cudaError_t launch_dense_ablation(const KernelParams& kp, dim3 grid, cudaStream_t s);

// Generic-taps kernel (sobel5_stream.cuh).
cudaError_t launch_generic(const KernelParams& kp, dim3 grid, int pf, bool default_taps,
                           MagMode mag, cudaStream_t s);

// Extra options of a launch beyond the plain StreamResult planes.
struct LaunchExtra {
    int pad = 0;                               // fused pad_replicate(img, 2)
    sobel5_minmax* minmax = nullptr;           // normalize pass 1
    const sobel5_norm_table* norm = nullptr;   // normalize pass 2
    int u8_norm = 0;
    uint32_t* s32 = nullptr;                   // exact g^2 plane (normalize pass 1)
    int n16 = 0;                               // gx..gdt as int16 (host-path wire)
    int frame0 = 0, row0 = 0;                  // the launch's place in the caller's
                                               // image (ParityViolation order key)
};

// The int16 D2H wire of the host path (sobel5_ctx.cu) applies: default taps
// on the packed kernel (every gradient in [-2^15, 2^15)) and SOBEL5_WIRE16
// not 0.  launch_common accepts n16 only for plain images with exactly the
// StreamResult planes.
bool n16_wire_ok(const sobel5_taps* taps);
// Sign-extends n int16 into int32 (sobel5_wire.cpp: AVX2 streaming stores).
void widen_i16(int32_t* dst, const int16_t* src, size_t n);
// g = sqrt(sum of the np int16 rows' squares), n pixels (the wire without g)
void magnitude_i16(double* g, const int16_t* const* src, int np, size_t n);
// One wire row decoded: the np int16 rows widened into dst[p] (nullptr =
// skip) and, with g, the magnitude -- in one AVX-512 pass when every
// destination can be 64-byte aligned at one column, else widen + magnitude.
void decode_row_i16(int32_t* const* dst, double* g, const int16_t* const* src, int np, size_t n);

// sobel5_launch_band whose first output row is row0 of the caller's image
// (the multi-GPU bands: a global ParityViolation order key)
sobel5_status launch_band_at(const uint8_t* d_top, const uint8_t* d_in, const uint8_t* d_bot,
                             int64_t in_pitch, int width, int band_rows, const sobel5_taps* taps,
                             int prefetch, const sobel5_planes* d_out, sobel5_diag* d_diag,
                             void* stream, int row0);

// Common launch path (validation in the reference's order, geometry, kernel
// selection) for plain, batched, band and detect launches.
sobel5_status launch_common(const uint8_t* top, const uint8_t* mid, const uint8_t* bot,
                            int64_t in_pitch, int64_t in_frame_stride, int width, int mid_rows,
                            int frames, const sobel5_taps* taps, int prefetch,
                            const sobel5_planes* out, int64_t out_frame_stride,
                            sobel5_diag* diag, void* stream, const LaunchExtra& ex);

sobel5_status map_cuda(cudaError_t e);
int choose_band(int out_w, int out_h, int frames, bool narrow_only);  // output rows per CTA
sobel5_status check_planes(const sobel5_planes* o, int out_w);

// 3x3 operator (sobel3_packed.cuh, sobel3_k.cu).
sobel5_status sobel3_common(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                            int width, int height, int frames, int prefetch,
                            const sobel5_planes* out, int64_t out_frame_stride, void* stream,
                            const LaunchExtra& ex);
bool taps_default(const sobel5_taps* t);  // equal to make_stream_taps(1, 2, 6, 4)
bool taps_packed(const sobel5_taps* t);   // a packed kernel (exact integer S) serves these taps
void count_launch(int n = 1);

}  // namespace sobel5_b200
