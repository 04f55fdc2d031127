// sobel5_k_pad.cu -- instantiations of the packed default-taps kernel with
// pad_replicate(img, 2) fused into the loads (image_io.hpp:279-291): the
// detect path's same-size edge map (sobel5_cli.cpp:133).
#include "sobel5_internal.h"
#include "sobel5_packed.cuh"

namespace sobel5_b200 {

namespace {
template <int PF, int OUTS>
cudaError_t go(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    if (PF > 0 && kp.tma_load)  // band rows (clamped) by TMA (launch_common decides)
        return launch_kp(sobel5_packed_default_kernel<0, kGeomPadTma, OUTS>, grid, kCtaThreads, 0, s, kp);
    return launch_kp(sobel5_packed_default_kernel<PF, kGeomPad, OUTS>, grid, kCtaThreads, 0, s, kp);
}

template <int PF>
cudaError_t outs(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    switch (packed_out_set(kp)) {
        case kOutSR: return go<PF, kOutSR>(kp, grid, s);
        case kOutU8: return go<PF, kOutU8>(kp, grid, s);
        case kOutMinMax: return go<PF, kOutMinMax>(kp, grid, s);
        case kOutMinMax | kOutS32: return go<PF, kOutMinMax | kOutS32>(kp, grid, s);
        case kOutU8 | kOutNorm: return go<PF, kOutU8 | kOutNorm>(kp, grid, s);
        default: return go<PF, kOutRuntime>(kp, grid, s);
    }
}
}  // namespace

cudaError_t launch_packed_pad(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s) {
    return pf ? outs<1>(kp, grid, s) : outs<0>(kp, grid, s);
}

}  // namespace sobel5_b200
