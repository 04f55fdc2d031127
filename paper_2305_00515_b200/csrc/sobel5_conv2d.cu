// sobel5_conv2d.cu -- the oracle's dense valid-mode correlation with an
// arbitrary 5x5 or 3x3 integer kernel, on the device.
//
// Reference: conv2d_valid(const GrayPlane&, const Kernel5&) and the Kernel3
// overload (oracle.hpp:19-49): out(y, x) = sum_ij k(i, j) * img(y+i, x+j)
// (correlation, no flip), accumulated in int64 and cast to int32.  Two's
// complement arithmetic mod 2^32 is a ring homomorphism, so an int32
// wrapping accumulator gives the same int32 as the int64 sum's cast.
//
// Not the hot path (run_stream is): it serves the drop-in's oracle.hpp so a
// reference caller's verify flow (sobel5_cli.cpp:187-234) runs on the GPU
// too.  One CTA stages a (kRows + K - 1) x (kCols + K - 1) input tile in
// shared memory with coalesced 4-byte loads; each thread computes 4
// adjacent outputs of one row from a register window, taps from the
// kernel-parameter bank.
#include <cuda_runtime.h>

#include <cstdint>

#include "sobel5_gpu.h"
#include "sobel5_internal.h"

namespace {

constexpr int kCols = 128;  // output columns per CTA (32 threads x 4)
constexpr int kRows = 16;   // output rows per CTA (threads stride over them)
constexpr int kThreads = 256;

struct ConvParams {
    const uint8_t* in;
    int64_t in_pitch;
    int32_t* out[4];
    double* g;  // sobel5_4d's magnitude (NK == 4)
    int64_t out_pitch;
    int out_w, out_h;
    int32_t k[4][25];
};

// NK kernels of size K over the same staged tile; with NK == 4 and a
// non-NULL g also the magnitude of sobel5_4d (oracle.hpp:88-97):
// sqrt(gx*gx + gy*gy + gd*gd + gdt*gdt) in double, left to right, each
// product and sum rounded on its own (no FMA contraction), as the
// reference's x86-64 build evaluates it.
template <int K, int NK>
__global__ void __launch_bounds__(kThreads) conv2d_valid_kernel(const __grid_constant__ ConvParams p) {
    constexpr int kTileW = kCols + 8;  // >= kCols + K - 1, multiple of 4
    constexpr int kTileH = kRows + K - 1;
    __shared__ __align__(16) uint8_t tile[kTileH][kTileW];
    const int x0 = blockIdx.x * kCols, y0 = blockIdx.y * kRows;
    const int in_w = p.out_w + K - 1, in_h = p.out_h + K - 1;
    // stage the tile: one 32-bit word per thread and step (rows are 4-byte
    // aligned: in_pitch % 16 == 0 and x0 % 128 == 0); bytes past the image
    // edge are zero and never reach a valid output
    for (int i = threadIdx.x; i < kTileH * (kTileW / 4); i += kThreads) {
        const int r = i / (kTileW / 4), c = (i % (kTileW / 4)) * 4;
        const int y = y0 + r, x = x0 + c;
        uint32_t w = 0u;
        if (y < in_h && x < in_w) {
            const uint8_t* src = p.in + static_cast<int64_t>(y) * p.in_pitch + x;
            if (x + 3 < in_w) {
                w = *reinterpret_cast<const uint32_t*>(src);
            } else {
                for (int b = 0; b < in_w - x; ++b) w |= static_cast<uint32_t>(src[b]) << (8 * b);
            }
        }
        *reinterpret_cast<uint32_t*>(&tile[r][c]) = w;
    }
    __syncthreads();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int cx = tx * 4;
    for (int r = ty; r < kRows; r += kThreads / 32) {
        const int oy = y0 + r;
        if (oy >= p.out_h) break;
        uint32_t acc[NK][4] = {};
#pragma unroll
        for (int i = 0; i < K; ++i) {
            uint32_t win[4 + K - 1];
#pragma unroll
            for (int j = 0; j < 4 + K - 1; ++j) win[j] = tile[r + i][cx + j];
#pragma unroll
            for (int n = 0; n < NK; ++n)
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    const uint32_t kw = static_cast<uint32_t>(p.k[n][i * K + j]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[n][q] += kw * win[q + j];
                }
        }
        const int64_t o = static_cast<int64_t>(oy) * p.out_pitch + x0 + cx;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (x0 + cx + q >= p.out_w) break;
#pragma unroll
            for (int n = 0; n < NK; ++n)
                if (p.out[n]) p.out[n][o + q] = static_cast<int32_t>(acc[n][q]);
            if (NK == 4 && p.g) {
                double s = 0.0;
#pragma unroll
                for (int n = 0; n < 4; ++n) {
                    const double v = static_cast<double>(static_cast<int32_t>(acc[n][q]));
                    s = n == 0 ? __dmul_rn(v, v) : __dadd_rn(s, __dmul_rn(v, v));
                }
                p.g[o + q] = __dsqrt_rn(s);
            }
        }
    }
}

sobel5_status conv_launch(const uint8_t* d_in, int64_t in_pitch, int width, int height,
                          const int32_t* kernels, int ksize, int nk, int32_t* const outs[4],
                          double* g, int64_t out_pitch, void* stream) {
    if (ksize != 3 && ksize != 5) return SOBEL5_INVALID_ARG;
    // oracle.hpp:20-22 / :36-38: size first
    if (width < ksize || height < ksize) return SOBEL5_IMAGE_TOO_SMALL;
    if (!d_in || !kernels) return SOBEL5_INVALID_ARG;
    if (in_pitch < width || in_pitch % 16 != 0 || reinterpret_cast<uintptr_t>(d_in) % 16 != 0)
        return SOBEL5_INVALID_ARG;
    const int out_w = width - ksize + 1, out_h = height - ksize + 1;
    if (out_pitch < out_w) return SOBEL5_INVALID_ARG;
    ConvParams p{};
    p.in = d_in;
    p.in_pitch = in_pitch;
    for (int n = 0; n < nk; ++n) {
        p.out[n] = outs[n];
        for (int i = 0; i < ksize * ksize; ++i) p.k[n][i] = kernels[n * ksize * ksize + i];
    }
    p.g = g;
    p.out_pitch = out_pitch;
    p.out_w = out_w;
    p.out_h = out_h;
    const dim3 grid(static_cast<unsigned>((out_w + kCols - 1) / kCols),
                    static_cast<unsigned>((out_h + kRows - 1) / kRows));
    if (grid.y > 65535u) return SOBEL5_INVALID_ARG;
    sobel5_b200::count_launch(1);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (nk == 4) conv2d_valid_kernel<5, 4><<<grid, kThreads, 0, s>>>(p);
    else if (ksize == 5) conv2d_valid_kernel<5, 1><<<grid, kThreads, 0, s>>>(p);
    else conv2d_valid_kernel<3, 1><<<grid, kThreads, 0, s>>>(p);
    return sobel5_b200::map_cuda(cudaGetLastError());
}

}  // namespace

extern "C" sobel5_status sobel5_conv2d_valid(const uint8_t* d_in, int64_t in_pitch, int width,
                                             int height, const int32_t* kernel, int ksize,
                                             int32_t* d_out, int64_t out_pitch, void* stream) {
    if (!d_out && width >= ksize && height >= ksize) return SOBEL5_INVALID_ARG;
    int32_t* const outs[4] = {d_out, nullptr, nullptr, nullptr};
    return conv_launch(d_in, in_pitch, width, height, kernel, ksize, 1, outs, nullptr, out_pitch,
                       stream);
}

extern "C" sobel5_status sobel5_dense_4d(const uint8_t* d_in, int64_t in_pitch, int width,
                                         int height, const int32_t* kernels,
                                         const sobel5_planes* d_out, void* stream) {
    if (!d_out && width >= 5 && height >= 5) return SOBEL5_INVALID_ARG;
    if (d_out && (d_out->g32 || d_out->u8)) return SOBEL5_INVALID_ARG;
    int32_t* const outs[4] = {d_out ? d_out->gx : nullptr, d_out ? d_out->gy : nullptr,
                              d_out ? d_out->gd : nullptr, d_out ? d_out->gdt : nullptr};
    return conv_launch(d_in, in_pitch, width, height, kernels, 5, 4, outs,
                       d_out ? d_out->g : nullptr, d_out ? d_out->pitch : 0, stream);
}
