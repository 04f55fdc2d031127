// sobel5_k_f32.cu -- instantiations of the packed-FP32 runtime-taps kernel
// (sobel5_f32x2.cuh) for every geometry, prefetch mode and magnitude mode.
#include "sobel5_f32x2.cuh"
#include "sobel5_internal.h"

namespace sobel5_b200 {

namespace {
template <int PF, int GEOM, int OUTS>
cudaError_t go2(const KernelParams& kp, dim3 grid, MagMode mag, cudaStream_t s) {
    // every value is below 2^22, so S < 2^46: exact in uint64 (kMagU64)
    if (mag == kMagU32)
        return launch_kp(sobel5_f32x2_kernel<PF, GEOM, kMagU32, OUTS>, grid, kCtaThreads, 0, s, kp);
    return launch_kp(sobel5_f32x2_kernel<PF, GEOM, kMagU64, OUTS>, grid, kCtaThreads, 0, s, kp);
}

template <int PF, int GEOM>
cudaError_t go(const KernelParams& kp, dim3 grid, MagMode mag, cudaStream_t s) {
    const bool sr = kp.gx && kp.gy && kp.gd && kp.gdt && kp.g && !kp.g32 && !kp.u8 &&
                    !kp.minmax && !kp.s32;
    return sr ? go2<PF, GEOM, kOutSR>(kp, grid, mag, s) : go2<PF, GEOM, kOutRuntime>(kp, grid, mag, s);
}

template <int PF>
cudaError_t geom(const KernelParams& kp, dim3 grid, MagMode mag, cudaStream_t s) {
    if (kp.pad) return go<PF, kGeomPad>(kp, grid, mag, s);
    if (kp.top_rows > 0 || kp.bot != nullptr) return go<PF, kGeomSeg>(kp, grid, mag, s);
    // band rows by TMA (launch_common decides), read from shared memory when consumed
    if (PF > 0 && kp.tma_load) return go<0, kGeomPlainTma>(kp, grid, mag, s);
    return go<PF, kGeomPlain>(kp, grid, mag, s);
}
}  // namespace

cudaError_t launch_f32(const KernelParams& kp, dim3 grid, int pf, MagMode mag, cudaStream_t s) {
    return pf ? geom<1>(kp, grid, mag, s) : geom<0>(kp, grid, mag, s);
}

}  // namespace sobel5_b200
