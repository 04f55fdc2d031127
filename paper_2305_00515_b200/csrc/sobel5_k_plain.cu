// sobel5_k_plain.cu -- instantiations of the packed default-taps kernel for
// plain images and batches (valid mode), one per output contract.
#include "sobel5_internal.h"
#include "sobel5_packed.cuh"

namespace sobel5_b200 {

namespace {
template <int PF, int OUTS>
cudaError_t go(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    // band rows by TMA (launch_common decides).  With the rows already in
    // shared memory the kernel reads each one when it is consumed
    // (instantiated with PF = 0): no register ring, 112 instead of 118
    // registers, 134.1 vs 134.9 us at 8K (profiles/r1/tma_load.txt).
    if constexpr (OUTS == kOutSR) {
        if (PF > 0 && kp.tma_load && kp.tstore == 2) {
            static const cudaError_t attr = cudaFuncSetAttribute(
                sobel5_packed_default_kernel<0, kGeomPlainTmaTw, kOutSR>,
                cudaFuncAttributeMaxDynamicSharedMemorySize, kTsSmemBytes);
            if (attr != cudaSuccess) return attr;
            return launch_kp(sobel5_packed_default_kernel<0, kGeomPlainTmaTw, kOutSR>, grid, kCtaThreads, kTsSmemBytes, s, kp);
        }
        if (PF > 0 && kp.tma_load && kp.tstore) {
            // StreamResult through TMA tensor stores (staging in dynamic smem)
            static const cudaError_t attr = cudaFuncSetAttribute(
                sobel5_packed_default_kernel<0, kGeomPlainTmaTs, kOutSR>,
                cudaFuncAttributeMaxDynamicSharedMemorySize, kTsSmemBytes);
            if (attr != cudaSuccess) return attr;
            return launch_kp(sobel5_packed_default_kernel<0, kGeomPlainTmaTs, kOutSR>, grid, kCtaThreads, kTsSmemBytes, s, kp);
        }
    }
    if (PF > 0 && kp.tma_load)
        return launch_kp(sobel5_packed_default_kernel<0, kGeomPlainTma, OUTS>, grid, kCtaThreads, 0, s, kp);
    return launch_kp(sobel5_packed_default_kernel<PF, kGeomPlain, OUTS>, grid, kCtaThreads, 0, s, kp);
}

template <int PF>
cudaError_t outs(const KernelParams& kp, dim3 grid, cudaStream_t s) {
    // compile-time output sets for the common contracts, runtime otherwise
    switch (packed_out_set(kp)) {
        case kOutSR: return go<PF, kOutSR>(kp, grid, s);
        case kOutSR | kOutN16: return go<PF, kOutSR | kOutN16>(kp, grid, s);
        case 15 | kOutN16: return go<PF, 15 | kOutN16>(kp, grid, s);
        case kOutSR | kOutU8: return go<PF, kOutSR | kOutU8>(kp, grid, s);
        case kOutU8: return go<PF, kOutU8>(kp, grid, s);
        case 15 | kOutG32: return go<PF, 15 | kOutG32>(kp, grid, s);
        case kOutMinMax: return go<PF, kOutMinMax>(kp, grid, s);
        case kOutMinMax | kOutS32: return go<PF, kOutMinMax | kOutS32>(kp, grid, s);
        case kOutU8 | kOutNorm: return go<PF, kOutU8 | kOutNorm>(kp, grid, s);
        default: return go<PF, kOutRuntime>(kp, grid, s);
    }
}
}  // namespace

cudaError_t launch_packed_plain(const KernelParams& kp, dim3 grid, int pf, cudaStream_t s) {
    return pf ? outs<1>(kp, grid, s) : outs<0>(kp, grid, s);
}

}  // namespace sobel5_b200
