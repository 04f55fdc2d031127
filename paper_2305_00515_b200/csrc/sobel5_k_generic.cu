// sobel5_k_generic.cu -- instantiations of the generic-taps kernel (any
// StreamTaps, including fault-injected ones; sobel5_stream.cuh).
#include "sobel5_internal.h"

namespace sobel5_b200 {

namespace {
template <int PF, class TAPS, int MAG>
cudaError_t go(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    if (kp.pad)
        return launch_kp(sobel5_stream_kernel<PF, TAPS, MAG, true>, grid, kCtaThreads, 0, s, kp);
    return launch_kp(sobel5_stream_kernel<PF, TAPS, MAG, false>, grid, kCtaThreads, 0, s, kp);
}

template <int PF>
cudaError_t pick(const KernelParams& kp, dim3 grid, bool dflt, MagMode mag, cudaStream_t s) {
    if (dflt) return go<PF, DefaultTaps, kMagU32>(kp, grid, s);
    if (mag == kMagU32) return go<PF, KernelParams, kMagU32>(kp, grid, s);
    return go<PF, KernelParams, kMagF64>(kp, grid, s);
}
}  // namespace

cudaError_t launch_generic(const KernelParams& kp, dim3 grid, int pf, bool default_taps,
                           MagMode mag, cudaStream_t s) {
    return pf ? pick<1>(kp, grid, default_taps, mag, s) : pick<0>(kp, grid, default_taps, mag, s);
}

}  // namespace sobel5_b200
