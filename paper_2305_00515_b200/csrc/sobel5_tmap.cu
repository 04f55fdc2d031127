// sobel5_tmap.cu -- host side of the tensor-map (TMA) stores of the
// StreamResult planes (sobel5_packed.cuh, kGeomPlainTmaTs): one CUtensorMap
// per plane, encoded with the driver's cuTensorMapEncodeTiled (fetched with
// cudaGetDriverEntryPoint, no -lcuda), cached per thread for repeated calls
// on the same buffers.
//
// The int32 planes are described as uint64 tensors of width ceil(out_w / 2)
// so that one box row is 256 elements = 512 int32 columns = a whole CTA tile
// (the box limit is 256 elements); for odd out_w the store writes one int32
// past out_w, inside the row pitch (pitch % 4 == 0, so pitch > out_w then).
// The g plane (float64) takes two 256-column boxes per CTA tile.  Rows past
// out_h / columns past the tensor width are clipped by the TMA unit.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstring>

#include "sobel5_internal.h"
#include "sobel5_packed.cuh"

namespace sobel5_b200 {

namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeFn>(nullptr);
        return reinterpret_cast<EncodeFn>(p);
    }();
    return fn;
}

bool encode(CUtensorMap* m, CUtensorMapDataType dt, void* base, uint64_t w, uint64_t h, uint64_t f,
            uint64_t row_bytes, uint64_t frame_bytes, uint32_t box_w, uint32_t box_h) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {w, h, f};
    const cuuint64_t strides[2] = {row_bytes, frame_bytes};
    const cuuint32_t box[3] = {box_w, box_h, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, dt, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Entry {
    const void* ptr[5];
    int out_w, out_h, frames, rows, box_cols;
    int64_t pitch, fstride;
    CUtensorMap map[5];
    bool valid;
};

}  // namespace

bool build_store_maps(KernelParams& kp, int frames, int rows, int box_cols) {
    if (!kp.gx || !kp.gy || !kp.gd || !kp.gdt || !kp.g) return false;
    const int64_t fstride = frames > 1 ? kp.out_frame_stride : kp.pitch * kp.out_h;
    if ((kp.pitch * 4) % 16 != 0 || (fstride * 4) % 16 != 0) return false;
    const void* ptr[5] = {kp.gx, kp.gy, kp.gd, kp.gdt, kp.g};
    thread_local Entry cache[4] = {};
    thread_local int next = 0;
    for (Entry& e : cache) {
        if (e.valid && std::memcmp(e.ptr, ptr, sizeof ptr) == 0 && e.out_w == kp.out_w &&
            e.out_h == kp.out_h && e.frames == frames && e.rows == rows && e.box_cols == box_cols && e.pitch == kp.pitch &&
            e.fstride == fstride) {
            std::memcpy(kp.tmap, e.map, sizeof kp.tmap);
            return true;
        }
    }
    Entry e{};
    std::memcpy(e.ptr, ptr, sizeof ptr);
    e.out_w = kp.out_w;
    e.out_h = kp.out_h;
    e.frames = frames;
    e.rows = rows;
    e.box_cols = box_cols;
    e.pitch = kp.pitch;
    e.fstride = fstride;
    const uint64_t w2 = (static_cast<uint64_t>(kp.out_w) + 1) / 2;
    void* ints[4] = {kp.gx, kp.gy, kp.gd, kp.gdt};
    for (int i = 0; i < 4; ++i)
        if (!encode(&e.map[i], CU_TENSOR_MAP_DATA_TYPE_UINT64, ints[i], w2, kp.out_h, frames,
                    kp.pitch * 4, fstride * 4, box_cols / 2, rows))
            return false;
    if (!encode(&e.map[4], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, kp.g, kp.out_w, kp.out_h, frames,
                kp.pitch * 8, fstride * 8, std::min(box_cols, 256), rows))
        return false;
    e.valid = true;
    cache[next] = e;
    next = (next + 1) % 4;
    std::memcpy(kp.tmap, e.map, sizeof kp.tmap);
    return true;
}

}  // namespace sobel5_b200
