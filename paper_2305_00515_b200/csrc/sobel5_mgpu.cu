// sobel5_mgpu.cu -- one image row-band partitioned over several GPUs from ONE
// process (BASELINE config C5; SURVEY.md sections 5 and 8e), behind the C
// ABI, plus the stream-ordered flag primitives the cross-process partition
// (paper_2305_00515_b200/bands.py) uses.
//
// The reference has no device decomposition; its parallel dispatcher is the
// strip thread pool run_strips_parallel (pipeline.hpp:416-445).  Here band k
// of N owns input rows [k*H/N, (k+1)*H/N) on devices[k] and writes the
// output rows whose 5x5 window is centred in it.  The 2 rows above and below
// a band (the 2r = 4-row vertical halo) come from the neighbours:
//
//   peer : the band kernel (sobel5_launch_band, kGeomSeg[Tma]) reads the
//          neighbour's rows straight from its HBM over NVLink / NVSwitch --
//          the exchange is fused into the stencil, no copy, no collective;
//   copy : interior rows first, then the 2-row halos copied device to device
//          (cudaMemcpyPeerAsync, overlapping the interior), then the two
//          2-row seams.
//
// Ordering is stream/event based, one stream per band, no host barrier:
// "ready[k]" is recorded on band k's stream when run_bands is called (all
// work enqueued on that stream before, e.g. the upload of its rows, is
// done), each band waits for its neighbours' ready events before reading
// their rows, records "done[k]" after its kernels, and at the end every band
// stream waits for its neighbours' done events -- so whatever the caller
// enqueues next on band k's stream (new input rows) runs only after every
// kernel that reads band k's rows has finished.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "sobel5_gpu.h"
#include "sobel5_internal.h"

namespace {

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

constexpr size_t kElem[7] = {4, 4, 4, 4, 8, 4, 1};  // gx gy gd gdt g g32 u8

struct Band {
    int device = 0;
    int r0 = 0, r1 = 0;        // input rows held
    int c0 = 0, c1 = 0;        // centre rows computed (image rows)
    cudaStream_t stream = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
    uint8_t* d_in = nullptr;   // body rows, pitch bytes
    uint8_t* d_halo = nullptr; // copy transport: 2 rows above + 2 rows below
    void* d_plane[7] = {};     // run_host: this band's output rows
    size_t d_plane_bytes[7] = {};
    sobel5_diag* d_diag = nullptr;  // run_host: recover_diag parity record
    int rows() const { return r1 - r0; }
};

// ---- driver entry points for stream memory operations (no libcuda link) ----
using PfnWait = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PfnWrite = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PfnWait g_wait = nullptr;
PfnWrite g_write = nullptr;
std::once_flag g_memop_once;

bool load_memops() {
    std::call_once(g_memop_once, [] {
        void* w = nullptr;
        void* r = nullptr;
        cudaDriverEntryPointQueryResult q1{}, q2{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess)
            g_wait = reinterpret_cast<PfnWait>(w);
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &r, cudaEnableDefault, &q2) == cudaSuccess &&
            q2 == cudaDriverEntryPointSuccess)
            g_write = reinterpret_cast<PfnWrite>(r);
        cudaGetLastError();
    });
    return g_wait && g_write;
}

}  // namespace

struct sobel5_mgpu {
    int width = 0, height = 0, transport = 0;
    int64_t in_pitch = 0;
    std::vector<Band> bands;
    sobel5_diag last_diag{};  // run_host's first parity violation
    int strip_w = 0;          // orders that pair (sobel5_mgpu_set_strip_width)
    sobel5_diag diag_init{};  // what each band's record starts from
};

namespace {

sobel5_status ck(cudaError_t e) { return sobel5_b200::map_cuda(e); }

#define CKS(expr)                                         \
    do {                                                  \
        const sobel5_status s_ = ck(expr);                \
        if (s_ != SOBEL5_OK) return s_;                   \
    } while (0)

sobel5_planes offset_planes(const sobel5_planes& p, int64_t rows) {
    sobel5_planes q = p;
    const int64_t off = rows * p.pitch;
    if (q.gx) q.gx += off;
    if (q.gy) q.gy += off;
    if (q.gd) q.gd += off;
    if (q.gdt) q.gdt += off;
    if (q.g) q.g += off;
    if (q.g32) q.g32 += off;
    if (q.u8) q.u8 += off;
    return q;
}

// Enqueues band k's kernels on its stream (after waiting for its
// neighbours' ready events).  `out` is the band's planes on its device.
sobel5_status run_band(sobel5_mgpu* m, int k, const sobel5_taps* taps, int prefetch,
                       const sobel5_planes& out, sobel5_diag* diag) {
    Band& b = m->bands[static_cast<size_t>(k)];
    const int n = static_cast<int>(m->bands.size());
    const bool has_top = k > 0, has_bot = k < n - 1;
    CKS(cudaSetDevice(b.device));
    if (has_top) CKS(cudaStreamWaitEvent(b.stream, m->bands[static_cast<size_t>(k - 1)].ready, 0));
    if (has_bot) CKS(cudaStreamWaitEvent(b.stream, m->bands[static_cast<size_t>(k + 1)].ready, 0));
    const int64_t P = m->in_pitch;
    if (m->transport == SOBEL5_MGPU_PEER || (!has_top && !has_bot)) {
        const uint8_t* top = nullptr;
        const uint8_t* bot = nullptr;
        if (has_top) {
            const Band& u = m->bands[static_cast<size_t>(k - 1)];
            top = u.d_in + static_cast<int64_t>(u.rows() - 2) * P;
        }
        if (has_bot) bot = m->bands[static_cast<size_t>(k + 1)].d_in;
        return sobel5_b200::launch_band_at(top, b.d_in, bot, P, m->width, b.rows(), taps, prefetch,
                                           &out, diag, b.stream, b.c0 - 2);
    }
    // copy transport: interior first (no halo needed), halos, then the seams
    const int top_rows = has_top ? 2 : 0;
    if (b.rows() > 4) {
        const sobel5_planes o = offset_planes(out, top_rows);
        if (sobel5_status st = sobel5_b200::launch_band_at(nullptr, b.d_in, nullptr, P, m->width,
                                                           b.rows(), taps, prefetch, &o, diag,
                                                           b.stream, b.c0 - 2 + top_rows);
            st != SOBEL5_OK)
            return st;
    }
    uint8_t* h_top = b.d_halo;
    uint8_t* h_bot = b.d_halo + 2 * P;
    if (has_top) {
        const Band& u = m->bands[static_cast<size_t>(k - 1)];
        CKS(cudaMemcpyPeerAsync(h_top, b.device, u.d_in + static_cast<int64_t>(u.rows() - 2) * P,
                                u.device, static_cast<size_t>(2 * P), b.stream));
    }
    if (has_bot) {
        const Band& d = m->bands[static_cast<size_t>(k + 1)];
        CKS(cudaMemcpyPeerAsync(h_bot, b.device, d.d_in, d.device, static_cast<size_t>(2 * P),
                                b.stream));
    }
    if (has_top) {  // centres r0, r0 + 1 from [halo; body rows 0..3]
        if (sobel5_status st = sobel5_b200::launch_band_at(h_top, b.d_in, nullptr, P, m->width, 4,
                                                           taps, prefetch, &out, diag, b.stream,
                                                           b.c0 - 2);
            st != SOBEL5_OK)
            return st;
    }
    if (has_bot) {  // centres r1 - 2, r1 - 1 from [body rows r1-4..r1-1; halo]
        const sobel5_planes o = offset_planes(out, b.c1 - b.c0 - 2);
        if (sobel5_status st = sobel5_b200::launch_band_at(
                nullptr, b.d_in + static_cast<int64_t>(b.rows() - 4) * P, h_bot, P, m->width, 4,
                taps, prefetch, &o, diag, b.stream, b.c1 - 4);
            st != SOBEL5_OK)
            return st;
    }
    return SOBEL5_OK;
}

}  // namespace

extern "C" {

sobel5_status sobel5_mgpu_create(sobel5_mgpu** out, const int* devices, int n, int width,
                                 int height, int transport) {
    if (!out) return SOBEL5_INVALID_ARG;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return SOBEL5_NO_DEVICE;
    }
    if (width < 5 || height < 5) return SOBEL5_IMAGE_TOO_SMALL;  // pipeline.hpp:454-456
    if (!devices || n < 1 || n > 64) return SOBEL5_INVALID_ARG;
    if (height < 4 * n) return SOBEL5_DIM_MISMATCH;  // every band needs >= 4 rows
    if (transport != SOBEL5_MGPU_AUTO && transport != SOBEL5_MGPU_PEER &&
        transport != SOBEL5_MGPU_COPY)
        return SOBEL5_INVALID_ARG;
    for (int k = 0; k < n; ++k)
        if (devices[k] < 0 || devices[k] >= ndev) return SOBEL5_INVALID_ARG;
    auto* m = new sobel5_mgpu;
    m->width = width;
    m->height = height;
    m->in_pitch = round_up(width, 128);
    m->bands.resize(static_cast<size_t>(n));
    // peer transport needs load access to each neighbour's memory
    bool peer_ok = true;
    for (int k = 0; k < n; ++k)
        for (int j : {k - 1, k + 1}) {
            if (j < 0 || j >= n || devices[j] == devices[k]) continue;
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, devices[k], devices[j]) != cudaSuccess || !can)
                peer_ok = false;
        }
    cudaGetLastError();
    if (transport == SOBEL5_MGPU_PEER && !peer_ok) {
        delete m;
        return SOBEL5_INVALID_ARG;
    }
    m->transport = transport == SOBEL5_MGPU_AUTO ? (peer_ok ? SOBEL5_MGPU_PEER : SOBEL5_MGPU_COPY)
                                                 : transport;
    sobel5_status st = SOBEL5_OK;
    for (int k = 0; k < n && st == SOBEL5_OK; ++k) {
        Band& b = m->bands[static_cast<size_t>(k)];
        b.device = devices[k];
        b.r0 = static_cast<int>(static_cast<int64_t>(k) * height / n);
        b.r1 = static_cast<int>(static_cast<int64_t>(k + 1) * height / n);
        b.c0 = std::max(b.r0, 2);
        b.c1 = std::min(b.r1, height - 2);
        st = ck(cudaSetDevice(b.device));
        if (st == SOBEL5_OK && m->transport == SOBEL5_MGPU_PEER)
            for (int j : {k - 1, k + 1}) {
                if (j < 0 || j >= n || devices[j] == b.device) continue;
                const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (e != cudaSuccess) st = ck(e);
            }
        if (st == SOBEL5_OK) st = ck(cudaStreamCreateWithFlags(&b.stream, cudaStreamNonBlocking));
        if (st == SOBEL5_OK) st = ck(cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming));
        if (st == SOBEL5_OK) st = ck(cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming));
        if (st == SOBEL5_OK)
            st = ck(cudaMalloc(reinterpret_cast<void**>(&b.d_in),
                               static_cast<size_t>(m->in_pitch) * b.rows()));
        if (st == SOBEL5_OK && m->transport == SOBEL5_MGPU_COPY)
            st = ck(cudaMalloc(reinterpret_cast<void**>(&b.d_halo),
                               static_cast<size_t>(m->in_pitch) * 4));
    }
    if (st != SOBEL5_OK) {
        sobel5_mgpu_destroy(m);
        return st;
    }
    *out = m;
    return SOBEL5_OK;
}

void sobel5_mgpu_destroy(sobel5_mgpu* m) {
    if (!m) return;
    for (Band& b : m->bands) {
        if (cudaSetDevice(b.device) != cudaSuccess) continue;
        if (b.stream) cudaStreamSynchronize(b.stream);
    }
    for (Band& b : m->bands) {
        if (cudaSetDevice(b.device) != cudaSuccess) continue;
        if (b.d_in) cudaFree(b.d_in);
        if (b.d_halo) cudaFree(b.d_halo);
        if (b.d_diag) cudaFree(b.d_diag);
        for (void* p : b.d_plane)
            if (p) cudaFree(p);
        if (b.ready) cudaEventDestroy(b.ready);
        if (b.done) cudaEventDestroy(b.done);
        if (b.stream) cudaStreamDestroy(b.stream);
    }
    cudaGetLastError();
    delete m;
}

sobel5_status sobel5_mgpu_band(const sobel5_mgpu* m, int k, sobel5_band_info* info) {
    if (!m || !info || k < 0 || k >= static_cast<int>(m->bands.size())) return SOBEL5_INVALID_ARG;
    const Band& b = m->bands[static_cast<size_t>(k)];
    info->device = b.device;
    info->r0 = b.r0;
    info->r1 = b.r1;
    info->out_row0 = b.c0 - 2;
    info->out_rows = b.c1 - b.c0;
    info->d_in = b.d_in;
    info->in_pitch = m->in_pitch;
    info->stream = b.stream;
    info->transport = m->transport;
    return SOBEL5_OK;
}

sobel5_status sobel5_mgpu_upload(sobel5_mgpu* m, const uint8_t* h_img) {
    if (!m || !h_img) return SOBEL5_INVALID_ARG;
    for (Band& b : m->bands) {
        CKS(cudaSetDevice(b.device));
        CKS(cudaMemcpy2DAsync(b.d_in, static_cast<size_t>(m->in_pitch),
                              h_img + static_cast<int64_t>(b.r0) * m->width,
                              static_cast<size_t>(m->width), static_cast<size_t>(m->width),
                              static_cast<size_t>(b.rows()), cudaMemcpyHostToDevice, b.stream));
    }
    return SOBEL5_OK;
}

sobel5_status sobel5_mgpu_synth(sobel5_mgpu* m, uint64_t seed, uint8_t mask) {
    if (!m) return SOBEL5_INVALID_ARG;
    for (Band& b : m->bands) {
        CKS(cudaSetDevice(b.device));
        if (sobel5_status st = sobel5_synth_random_device(b.d_in, m->in_pitch, m->width, b.rows(),
                                                          b.r0, seed, mask, b.stream);
            st != SOBEL5_OK)
            return st;
    }
    return SOBEL5_OK;
}

}  // extern "C"

namespace {
sobel5_status run_bands_impl(sobel5_mgpu* m, const sobel5_taps* taps, int prefetch,
                             const sobel5_planes* d_out, bool with_diag) {
    const int n = static_cast<int>(m->bands.size());
    for (Band& b : m->bands) {  // everything enqueued so far on band k's stream
        CKS(cudaSetDevice(b.device));
        CKS(cudaEventRecord(b.ready, b.stream));
    }
    for (int k = 0; k < n; ++k) {
        sobel5_diag* dg = with_diag ? m->bands[static_cast<size_t>(k)].d_diag : nullptr;
        if (sobel5_status st = run_band(m, k, taps, prefetch, d_out[k], dg); st != SOBEL5_OK) return st;
        CKS(cudaEventRecord(m->bands[static_cast<size_t>(k)].done, m->bands[static_cast<size_t>(k)].stream));
    }
    // later writes to band k's rows (enqueued by the caller on its stream)
    // wait for every kernel that reads them
    for (int k = 0; k < n; ++k) {
        Band& b = m->bands[static_cast<size_t>(k)];
        CKS(cudaSetDevice(b.device));
        if (k > 0) CKS(cudaStreamWaitEvent(b.stream, m->bands[static_cast<size_t>(k - 1)].done, 0));
        if (k < n - 1) CKS(cudaStreamWaitEvent(b.stream, m->bands[static_cast<size_t>(k + 1)].done, 0));
    }
    return SOBEL5_OK;
}
}  // namespace

extern "C" {

sobel5_status sobel5_mgpu_run_bands(sobel5_mgpu* m, const sobel5_taps* taps, int prefetch,
                                    const sobel5_planes* d_out) {
    if (!m || !taps || !d_out) return SOBEL5_INVALID_ARG;
    return run_bands_impl(m, taps, prefetch, d_out, false);
}

sobel5_status sobel5_mgpu_sync(sobel5_mgpu* m) {
    if (!m) return SOBEL5_INVALID_ARG;
    for (Band& b : m->bands) {
        CKS(cudaSetDevice(b.device));
        CKS(cudaStreamSynchronize(b.stream));
    }
    return SOBEL5_OK;
}

sobel5_status sobel5_mgpu_run_host(sobel5_mgpu* m, const uint8_t* h_in, const sobel5_taps* taps,
                                   int prefetch, const sobel5_planes* h_out) {
    if (!m || !h_in || !taps || !h_out) return SOBEL5_INVALID_ARG;
    const int out_w = m->width - 4;
    if (h_out->pitch != out_w) return SOBEL5_INVALID_ARG;
    void* hp[7] = {h_out->gx, h_out->gy, h_out->gd, h_out->gdt, h_out->g, h_out->g32, h_out->u8};
    const int64_t dpitch = round_up(out_w, 32);
    std::vector<sobel5_planes> dp(m->bands.size());
    for (size_t k = 0; k < m->bands.size(); ++k) {
        Band& b = m->bands[k];
        CKS(cudaSetDevice(b.device));
        dp[k].pitch = dpitch;
        void** slots[7] = {reinterpret_cast<void**>(&dp[k].gx),  reinterpret_cast<void**>(&dp[k].gy),
                           reinterpret_cast<void**>(&dp[k].gd),  reinterpret_cast<void**>(&dp[k].gdt),
                           reinterpret_cast<void**>(&dp[k].g),   reinterpret_cast<void**>(&dp[k].g32),
                           reinterpret_cast<void**>(&dp[k].u8)};
        for (int i = 0; i < 7; ++i) {
            if (!hp[i]) continue;
            const size_t bytes = static_cast<size_t>(dpitch) * std::max(1, b.c1 - b.c0) * kElem[i];
            if (b.d_plane_bytes[i] < bytes) {
                if (b.d_plane[i]) cudaFree(b.d_plane[i]);
                b.d_plane[i] = nullptr;
                b.d_plane_bytes[i] = 0;
                CKS(cudaMalloc(&b.d_plane[i], bytes));
                b.d_plane_bytes[i] = bytes;
            }
            *slots[i] = b.d_plane[i];
        }
    }
    for (Band& b : m->bands) {
        CKS(cudaSetDevice(b.device));
        if (!b.d_diag) CKS(cudaMalloc(reinterpret_cast<void**>(&b.d_diag), sizeof(sobel5_diag)));
        m->diag_init = sobel5_diag{};
        m->diag_init.strip_w = m->strip_w;
        CKS(cudaMemcpyAsync(b.d_diag, &m->diag_init, sizeof(sobel5_diag), cudaMemcpyHostToDevice,
                            b.stream));
    }
    if (sobel5_status st = sobel5_mgpu_upload(m, h_in); st != SOBEL5_OK) return st;
    if (sobel5_status st = run_bands_impl(m, taps, prefetch, dp.data(), true); st != SOBEL5_OK)
        return st;
    for (size_t k = 0; k < m->bands.size(); ++k) {  // each band's rows over its own link
        Band& b = m->bands[k];
        CKS(cudaSetDevice(b.device));
        for (int i = 0; i < 7; ++i) {
            if (!hp[i]) continue;
            const size_t es = kElem[i];
            CKS(cudaMemcpy2DAsync(static_cast<char*>(hp[i]) + static_cast<size_t>(b.c0 - 2) * out_w * es,
                                  static_cast<size_t>(out_w) * es, b.d_plane[i],
                                  static_cast<size_t>(dpitch) * es, static_cast<size_t>(out_w) * es,
                                  static_cast<size_t>(b.c1 - b.c0), cudaMemcpyDeviceToHost, b.stream));
        }
    }
    if (sobel5_status st = sobel5_mgpu_sync(m); st != SOBEL5_OK) return st;
    // recover_diag (pipeline.hpp:268-273): the bands' keys are global (strip,
    // row, column), so the reported pair is the band record with the earliest
    // key (stored inverted: the largest), the count the sum over bands
    bool odd = false;
    sobel5_diag first{};
    int64_t total = 0;
    for (Band& b : m->bands) {
        sobel5_diag d{};
        CKS(cudaSetDevice(b.device));
        CKS(cudaMemcpy(&d, b.d_diag, sizeof d, cudaMemcpyDeviceToHost));
        if (!d.violations) continue;
        total += d.violations;
        if (!odd || d.order > first.order) first = d;
        odd = true;
    }
    if (!odd) return SOBEL5_OK;
    first.violations = static_cast<int32_t>(std::min<int64_t>(total, INT32_MAX));
    m->last_diag = first;
    return SOBEL5_PARITY_VIOLATION;
}

sobel5_status sobel5_mgpu_set_strip_width(sobel5_mgpu* m, int strip_w) {
    if (!m || strip_w < 0) return SOBEL5_INVALID_ARG;
    m->strip_w = strip_w;
    return SOBEL5_OK;
}

sobel5_status sobel5_mgpu_last_diag(const sobel5_mgpu* m, sobel5_diag* out) {
    if (!m || !out) return SOBEL5_INVALID_ARG;
    *out = m->last_diag;
    return SOBEL5_OK;
}

// ---- stream-ordered flags (cross-process ordering of the peer transport) ----

sobel5_status sobel5_host_register(void* p, size_t bytes, void** d_ptr) {
    if (!p || !bytes || !d_ptr) return SOBEL5_INVALID_ARG;
    CKS(cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    CKS(cudaHostGetDevicePointer(d_ptr, p, 0));
    return SOBEL5_OK;
}

sobel5_status sobel5_host_unregister(void* p) {
    if (!p) return SOBEL5_INVALID_ARG;
    return ck(cudaHostUnregister(p));
}

sobel5_status sobel5_stream_write_u32(uint32_t* d_flag, uint32_t value, void* stream) {
    if (!d_flag) return SOBEL5_INVALID_ARG;
    if (!load_memops()) return SOBEL5_CUDA_ERROR;
    return g_write(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(d_flag), value, 0) ==
                   CUDA_SUCCESS
               ? SOBEL5_OK
               : SOBEL5_CUDA_ERROR;
}

sobel5_status sobel5_stream_wait_u32(const uint32_t* d_flag, uint32_t value, void* stream) {
    if (!d_flag) return SOBEL5_INVALID_ARG;
    if (!load_memops()) return SOBEL5_CUDA_ERROR;
    return g_wait(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(d_flag), value,
                  CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS
               ? SOBEL5_OK
               : SOBEL5_CUDA_ERROR;
}

}  // extern "C"
