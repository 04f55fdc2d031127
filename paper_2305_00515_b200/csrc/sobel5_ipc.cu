// sobel5_ipc.cu -- CUDA IPC plumbing for the row-band partition (BASELINE
// config C5): each rank exports the device buffer holding its band, the
// neighbours map it, and sobel5_launch_band reads the 2-row halos straight
// from the peer mapping (NVLink / NVSwitch), so no separate halo exchange
// runs at all.  The band buffers may be sub-allocations (e.g. from PyTorch's
// caching allocator): the exported handle names the containing allocation
// and carries the byte offset of the pointer inside it.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <unordered_map>

#include "sobel5_gpu.h"

namespace {

std::mutex g_mu;
std::unordered_map<const void*, void*> g_mapped;  // user pointer -> mapped base

// cuMemGetAddressRange through the runtime's driver entry point, so the
// library does not link libcuda directly (it must load on CPU-only hosts).
using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range() {
    static AddrRangeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<AddrRangeFn>(p);
    }();
    return fn;
}

sobel5_status status_of(cudaError_t e) {
    if (e == cudaSuccess) return SOBEL5_OK;
    if (e == cudaErrorMemoryAllocation) return SOBEL5_OUT_OF_MEMORY;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return SOBEL5_NO_DEVICE;
    return SOBEL5_CUDA_ERROR;
}

}  // namespace

extern "C" {

sobel5_status sobel5_ipc_export(const void* d_ptr, sobel5_ipc_handle* out) {
    if (!d_ptr || !out) return SOBEL5_INVALID_ARG;
    CUdeviceptr base = 0;
    size_t size = 0;
    AddrRangeFn range = addr_range();
    if (!range) return SOBEL5_NO_DEVICE;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS)
        return SOBEL5_INVALID_ARG;
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return status_of(e);
    static_assert(sizeof(h) <= sizeof(out->bytes), "IPC handle size");
    std::memset(out, 0, sizeof *out);
    std::memcpy(out->bytes, &h, sizeof h);
    out->offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
    return SOBEL5_OK;
}

sobel5_status sobel5_ipc_import(const sobel5_ipc_handle* h, const void** d_ptr) {
    if (!h || !d_ptr) return SOBEL5_INVALID_ARG;
    cudaIpcMemHandle_t ch;
    std::memcpy(&ch, h->bytes, sizeof ch);
    void* base = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&base, ch, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return status_of(e);
    const void* p = static_cast<const char*>(base) + h->offset;
    std::lock_guard<std::mutex> lk(g_mu);
    g_mapped[p] = base;
    *d_ptr = p;
    return SOBEL5_OK;
}

sobel5_status sobel5_ipc_release(const void* d_ptr) {
    void* base = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_mapped.find(d_ptr);
        if (it == g_mapped.end()) return SOBEL5_INVALID_ARG;
        base = it->second;
        g_mapped.erase(it);
    }
    return status_of(cudaIpcCloseMemHandle(base));
}

}  // extern "C"
