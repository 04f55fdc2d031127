// sobel5_k_seg.cu -- instantiations of the packed default-taps kernel for
// row bands with halos (config C5), including halos read from a peer GPU.
#include "sobel5_internal.h"
#include "sobel5_packed.cuh"

namespace sobel5_b200 {

namespace {
template <int PF, int OUTS>
cudaError_t go(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    // band rows by TMA for the CTAs whose rows are all in the local band
    // (launch_common decides); the halo-touching CTAs load from global
    if (PF > 0 && kp.tma_load)
        return launch_kp(sobel5_packed_default_kernel<0, kGeomSegTma, OUTS>, grid, kCtaThreads, 0, s, kp);
    return launch_kp(sobel5_packed_default_kernel<PF, kGeomSeg, OUTS>, grid, kCtaThreads, 0, s, kp);
}

template <int PF>
cudaError_t outs(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    switch (packed_out_set(kp)) {
        case kOutSR: return go<PF, kOutSR>(kp, grid, s);
        case kOutU8: return go<PF, kOutU8>(kp, grid, s);
        default: return go<PF, kOutRuntime>(kp, grid, s);
    }
}
}  // namespace

cudaError_t launch_packed_seg(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s) {
    return pf ? outs<1>(kp, grid, s) : outs<0>(kp, grid, s);
}

}  // namespace sobel5_b200
