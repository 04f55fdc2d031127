// sobel5_k_rtaps.cu -- instantiations of the packed kernel with RUNTIME taps
// (any StreamTaps whose gx, gy, P and M responses fit int16: e.g. small
// FilterParams, or fault-injected defaults), for every geometry.
#include "sobel5_internal.h"
#include "sobel5_packed.cuh"

namespace sobel5_b200 {

namespace {
template <int PF, int GEOM, int OUTS>
cudaError_t go(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    return launch_kp(sobel5_packed_default_kernel<PF, GEOM, OUTS, true>, grid, kCtaThreads, 0, s, kp);
}

template <int PF, int GEOM>
cudaError_t outs(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    switch (packed_out_set(kp)) {
        case kOutSR: return go<PF, GEOM, kOutSR>(kp, grid, s);
        case kOutU8: return go<PF, GEOM, kOutU8>(kp, grid, s);
        case kOutMinMax | kOutS32: return go<PF, GEOM, kOutMinMax | kOutS32>(kp, grid, s);
        default: return go<PF, GEOM, kOutRuntime>(kp, grid, s);
    }
}
}  // namespace

cudaError_t launch_packed_rt_plain(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s) {
    return pf ? outs<1, kGeomPlain>(kp, grid, s) : outs<0, kGeomPlain>(kp, grid, s);
}
cudaError_t launch_packed_rt_seg(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s) {
    return pf ? outs<1, kGeomSeg>(kp, grid, s) : outs<0, kGeomSeg>(kp, grid, s);
}
cudaError_t launch_packed_rt_pad(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s) {
    return pf ? outs<1, kGeomPad>(kp, grid, s) : outs<0, kGeomPad>(kp, grid, s);
}

}  // namespace sobel5_b200
