// sobel5_ctx.cu -- device context and the host-buffer entry point that the
// C++ run_stream wrapper (include/sobel5_b200/sobel5.hpp) calls.
//
// The reference allocates five zero-filled output planes per call
// (pipeline.hpp:462-467) and walks strips on CPU threads (:416-445).  Here a
// context owns the device side once: pitched device planes cached across
// calls, three streams (H2D, compute, D2H) and per-chunk events, so the
// image is processed as row chunks whose upload, kernel and download
// overlap:
//
//   s_h2d : [in 0][in 1][in 2] ...
//   s_comp:       [k 0 ][k 1 ][k 2] ...        (waits on in k)
//   s_d2h :             [out 0    ][out 1 ]... (waits on k k)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "sobel5_gpu.h"
#include "sobel5_internal.h"

namespace {

// Host worker pool for the copies between pinned staging and caller memory
// and the int16 wire decode (one host thread moves ~14 GB/s; the decode's
// streaming stores reach ~112 GB/s with 16: profiles/r1/alloc_probe.txt,
// profiles/r2/wire_probe.txt).  The calling thread takes part.
class HostPool {
public:
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    // fn(i) for i in [0, n), returns when all are done
    void run(int n, const std::function<void(int)>& fn) {
        if (n <= 0) return;
        if (th_.empty()) start();
        auto b = std::make_shared<Batch>();
        b->fn = &fn;
        b->n = n;
        b->left = n;
        {
            std::lock_guard<std::mutex> g(m_);
            batch_ = b;
            ++gen_;
            gen_seen_.store(gen_, std::memory_order_release);
        }
        cv_.notify_all();
        work(*b);
        std::unique_lock<std::mutex> g(b->m);
        b->done.wait(g, [&] { return b->left == 0; });
    }
    int size() const { return static_cast<int>(th_.size()) + 1; }
    // threads including the caller, starting the pool if needed
    int threads() {
        if (th_.empty()) start();
        return size();
    }

private:
    // One run(): a worker that wakes late only sees next >= n and leaves
    // without touching fn (which may be gone by then).
    struct Batch {
        const std::function<void(int)>* fn = nullptr;
        int n = 0;
        std::atomic<int> next{0};
        int left = 0;
        std::mutex m;
        std::condition_variable done;
    };
    void start() {
        // threads incl. the caller: the host's cores shared by the node's
        // local ranks (LOCAL_WORLD_SIZE, set by torchrun), or
        // SOBEL5_HOST_THREADS.  The host path is bound by host memory
        // traffic, which scales with threads: 8K e2e 11.4-13.3 ms at 8, 9.1
        // at 16 on the 16-core B200 host (profiles/r2/host_threads.txt).
        const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
        const char* lw = std::getenv("LOCAL_WORLD_SIZE");
        const unsigned ranks = lw && *lw && std::atoi(lw) > 0 ? static_cast<unsigned>(std::atoi(lw)) : 1u;
        const char* v = std::getenv("SOBEL5_HOST_THREADS");
        const unsigned want = v && *v && std::atoi(v) > 0 ? static_cast<unsigned>(std::atoi(v))
                                                          : std::max(2u, hw / ranks);
        const int n = static_cast<int>(std::max(1u, std::min(want, hw)) - 1);
        for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
    }
    static void work(Batch& b) {
        int done = 0;
        for (int i; (i = b.next.fetch_add(1)) < b.n;) {
            (*b.fn)(i);
            ++done;
        }
        if (done) {
            std::lock_guard<std::mutex> g(b.m);
            b.left -= done;
            if (b.left == 0) b.done.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            // spin briefly before blocking: the host path hands out a batch
            // per row chunk every ~0.2 ms, and a futex wake-up of the whole
            // pool costs tens of microseconds per batch (SOBEL5_POOL_SPIN_US)
            const auto t0 = std::chrono::steady_clock::now();
            while (gen_seen_.load(std::memory_order_acquire) == seen &&
                   std::chrono::steady_clock::now() - t0 < spin_)
                spin_pause();
            std::shared_ptr<Batch> b;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                b = batch_;
            }
            if (b) work(*b);
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_;
    std::shared_ptr<Batch> batch_;
    uint64_t gen_ = 0;
    std::atomic<uint64_t> gen_seen_{0};
    std::chrono::microseconds spin_{[] {
        const char* v = std::getenv("SOBEL5_POOL_SPIN_US");
        return v && *v ? std::atoi(v) : 300;
    }()};
    bool stop_ = false;
    static void spin_pause() {
#if defined(__x86_64__) || defined(__i386__)
        __builtin_ia32_pause();
#endif
    }
};

}  // namespace

struct sobel5_ctx {
    int device = 0;
    cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
    uint8_t* d_in = nullptr;
    size_t d_in_bytes = 0;
    void* d_plane[7] = {};
    size_t d_plane_bytes[7] = {};
    sobel5_diag* d_diag = nullptr;
    sobel5_diag* h_diag = nullptr;  // pinned: [0] the call's result, [1] its initial value
    int strip_w = 0;                // sobel5_ctx_set_strip_width (ParityViolation order)
    uint64_t last_d2h = 0;          // bytes the last stream call moved device -> host
    void* d_scratch = nullptr;      // detect / normalize scratch
    size_t d_scratch_bytes = 0;
    // pinned staging: the input image and the planes bound for pageable memory
    void* h_in_stage = nullptr;
    size_t h_in_stage_bytes = 0;
    void* h_stage[7] = {};
    size_t h_stage_bytes[7] = {};
    // int16 wire (SOBEL5_WIRE16): gx gy gd gdt of the current call land here
    // as int16 and are widened into the int32 destinations (sobel5_wire.cpp)
    void* h_wire[4] = {};
    size_t h_wire_bytes[4] = {};
    bool wire = false;
    // sobel5_run_host's wire layout is chunk-major: chunk k's four int16
    // planes are one contiguous block (device and staging), moved by ONE
    // copy per chunk instead of four; wire_pitch = their row pitch (elements)
    bool wire_cm = false;
    int wire_np = 4;  // int16 planes on the wire: slots 0..wire_np-1 (4: 5x5, 2: 3x3 gx gy)
    // g is not on the chunk-major wire: the host rebuilds it from the int16
    // rows while widening them (sobel5_wire.cpp; SOBEL5_WIRE_G=0 ships it)
    bool wire_g = false;
    int64_t wire_pitch = 0;
    void* d_wire = nullptr;
    size_t d_wire_bytes = 0;
    // sobel5_run_host_frames: a ring of kFrameSlots units (frame row chunks)
    // in flight -- device input / output slots, pinned staging slots, events
    void* f_d_in = nullptr;
    size_t f_d_in_bytes = 0;
    void* f_d_out = nullptr;
    size_t f_d_out_bytes = 0;
    void* f_h_stage = nullptr;
    size_t f_h_stage_bytes = 0;
    std::vector<cudaEvent_t> f_ev;
    std::vector<cudaEvent_t> ev_in, ev_comp, ev_out;
    HostPool pool;
    // state between sobel5_run_host_begin and _finish
    struct Pending {
        bool active = false;
        int out_w = 0, out_h = 0, chunk = 0, n_chunks = 0;
        unsigned mask = 0;
        sobel5_status status = SOBEL5_OK;
    } pend;
    std::string last_error;
};

namespace {

constexpr size_t kElem[7] = {4, 4, 4, 4, 8, 4, 1};  // gx gy gd gdt g g32 u8

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// Zeroes the device diagnostics for a call, with the context's strip width
// (the ParityViolation order key) -- an H2D copy of h_diag[1] on s_comp.
cudaError_t reset_diag(sobel5_ctx* ctx) {
    ctx->h_diag[1] = sobel5_diag{};
    ctx->h_diag[1].strip_w = ctx->strip_w;
    return cudaMemcpyAsync(ctx->d_diag, &ctx->h_diag[1], sizeof(sobel5_diag), cudaMemcpyHostToDevice,
                           ctx->s_comp);
}

// bytes per element of plane slot i as it crosses PCIe in the current call
size_t wire_elem(const sobel5_ctx* ctx, int i) { return ctx->wire && i < ctx->wire_np ? 2 : kElem[i]; }

// The int16 wire applies to a 5x5 call with exactly the StreamResult planes
// and default taps (sobel5_b200::n16_wire_ok), if its int16 staging fits.
// The split begin/_chunk form (the C++ drop-in, which appends each row
// chunk into freshly allocated planes) uses it too, with 8 row chunks
// (8K run_stream 48.2-50.6 vs 53.4-54.5 ms without the wire; 16 chunks
// cost it ~10 ms of per-chunk synchronisation: profiles/r2/cpp_wire.txt).
// The 3x3 operator's Stream3Result (gx, gy, g; |gx|, |gy| <= 1020) rides it
// the same way with two int16 planes.
bool want_wire(unsigned mask, const sobel5_taps* taps, int op, bool /*split*/);

// With the chunk-major wire, g (a function of the int16 gradients alone) is
// rebuilt on the host unless SOBEL5_WIRE_G=0: 8 instead of 16 B/px over PCIe
// for the 5x5 StreamResult, 4 instead of 12 for the 3x3 one.
bool want_host_g() {
    const char* v = std::getenv("SOBEL5_WIRE_G");
    return !(v && *v && std::atoi(v) == 0);
}

// Rows [r0, r0 + rows) of one chunk-major wire block (plane p's row r at
// src + (p * plane_rows + r) * spitch): widened into the int32 planes dst[p]
// (rows of out_w, nullptr = not wanted) and, with g, the magnitude rebuilt.
void decode_wire_rows(void* const dst[7], const int16_t* src, int np, int64_t plane_rows,
                      int64_t spitch, int out_w, int64_t r0, int64_t rows, bool with_g) {
    for (int64_t r = r0; r < r0 + rows; ++r) {
        const int16_t* row[4] = {};
        int32_t* out[4] = {};
        for (int p = 0; p < np; ++p) {
            row[p] = src + (p * plane_rows + r) * spitch;
            if (dst[p]) out[p] = static_cast<int32_t*>(dst[p]) + r * out_w;
        }
        sobel5_b200::decode_row_i16(out, with_g ? static_cast<double*>(dst[4]) + r * out_w : nullptr,
                                    row, np, static_cast<size_t>(out_w));
    }
}

// Rows per decode piece of a wire chunk: ~1 MiB of output per piece
// (SOBEL5_DECODE_SPLIT=mib, default) or the rows split evenly over the pool
// (=pool).
int decode_rows_per_piece(sobel5_ctx* ctx, int rows, int out_w) {
    static const bool even = [] {
        const char* v = std::getenv("SOBEL5_DECODE_SPLIT");
        return v && std::strcmp(v, "pool") == 0;
    }();
    if (even) {
        const int nt = ctx->pool.threads();
        return std::max(1, (rows + nt - 1) / nt);
    }
    return std::max(1, (1 << 20) / (std::max(out_w, 1) * 24));
}

bool want_wire(unsigned mask, const sobel5_taps* taps, int op, bool /*split*/) {
    if (op == 3) {
        const char* v = std::getenv("SOBEL5_WIRE16");
        return mask == 0x13u && !(v && *v && std::atoi(v) == 0);
    }
    return op == 5 && mask == 0x1fu && sobel5_b200::n16_wire_ok(taps);
}

sobel5_status fail(sobel5_ctx* c, cudaError_t e) {
    c->last_error = cudaGetErrorString(e);
    if (e == cudaErrorMemoryAllocation) return SOBEL5_OUT_OF_MEMORY;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return SOBEL5_NO_DEVICE;
    return SOBEL5_CUDA_ERROR;
}

#define CK(expr)                                        \
    do {                                                \
        cudaError_t e_ = (expr);                        \
        if (e_ != cudaSuccess) return fail(ctx, e_);    \
    } while (0)

cudaError_t ensure(void** p, size_t* cap, size_t bytes) {
    if (*cap >= bytes) return cudaSuccess;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) *cap = bytes;
    return e;
}

cudaError_t ensure_host(void** p, size_t* cap, size_t bytes) {
    if (*cap >= bytes) return cudaSuccess;
    if (*p) cudaFreeHost(*p);
    *p = nullptr;
    *cap = 0;
    cudaError_t e = cudaMallocHost(p, bytes);
    if (e == cudaSuccess) *cap = bytes;
    return e;
}

cudaError_t ensure_events(std::vector<cudaEvent_t>& v, size_t n) {
    while (v.size() < n) {
        cudaEvent_t ev;
        cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
        v.push_back(ev);
    }
    return cudaSuccess;
}

// Pinned staging is cached per context up to this many bytes in total
// (SOBEL5_STAGING_MAX_MB, default 4096); planes beyond it are downloaded
// straight into pageable memory (the driver stages them, slower but bounded).
size_t staging_cap() {
    static const size_t cap = [] {
        const char* v = std::getenv("SOBEL5_STAGING_MAX_MB");
        return (v && *v ? static_cast<size_t>(std::atoll(v)) : size_t{4096}) << 20;
    }();
    return cap;
}

// Page-locked host memory (cudaMallocHost / cudaHostRegister) is DMA'd
// directly; anything else goes through the context's pinned staging.
bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Parallel memcpy of n bytes in >= 4 MiB pieces on the context's pool.
void par_copy(sobel5_ctx* ctx, void* dst, const void* src, size_t n) {
    constexpr size_t kPiece = size_t{4} << 20;
    const int pieces = static_cast<int>(std::min<size_t>(
        static_cast<size_t>(ctx->pool.size()) * 2, std::max<size_t>(1, n / kPiece)));
    if (pieces <= 1) {
        std::memcpy(dst, src, n);
        return;
    }
    const size_t per = (n + pieces - 1) / pieces;
    ctx->pool.run(pieces, [&](int i) {
        const size_t o = static_cast<size_t>(i) * per;
        if (o < n)
            std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                        std::min(per, n - o));
    });
}

// Pinned staging one host call may use (the SOBEL5_STAGING_MAX_MB cap counts
// the input and every plane of the call).  take(n) reserves n bytes if they
// fit; what does not fit is copied straight from / to pageable memory (the
// driver stages it: slower, but bounded).
struct StageBudget {
    size_t left = staging_cap();
    bool take(size_t n) {
        if (n > left) return false;
        left -= n;
        return true;
    }
};

// A pageable input is first copied into pinned staging (in parallel) so the
// uploads that follow are true asynchronous DMA; *src is what to upload.
// Without room in the budget it is uploaded from pageable memory directly.
sobel5_status stage_input(sobel5_ctx* ctx, const uint8_t* h_in, size_t n, const uint8_t** src,
                          StageBudget& budget) {
    *src = h_in;
    if (is_pinned(h_in) || !budget.take(n)) return SOBEL5_OK;
    CK(ensure_host(&ctx->h_in_stage, &ctx->h_in_stage_bytes, n));
    par_copy(ctx, ctx->h_in_stage, h_in, n);
    *src = static_cast<const uint8_t*>(ctx->h_in_stage);
    return SOBEL5_OK;
}

// Enqueues the download of `rows` rows of plane slot i (device pitch dpitch
// elements) to tightly packed host memory: straight into a pinned dst, or
// into the pinned staging h_stage[i], recorded in *staged for
// finish_staged() once the stream has synchronised (pageable destinations
// beyond the staging budget are written by the driver directly).
sobel5_status download_plane(sobel5_ctx* ctx, int i, void* dst, const void* d_src, int out_w,
                             int rows, int64_t dpitch, cudaStream_t s, void* staged[7],
                             StageBudget& budget) {
    const size_t es = kElem[i], row = static_cast<size_t>(out_w) * es;
    void* to = dst;
    if (!is_pinned(dst) && budget.take(row * rows)) {
        CK(ensure_host(&ctx->h_stage[i], &ctx->h_stage_bytes[i], row * rows));
        to = ctx->h_stage[i];
        staged[i] = dst;
    }
    CK(cudaMemcpy2DAsync(to, row, d_src, static_cast<size_t>(dpitch) * es, row,
                         static_cast<size_t>(rows), cudaMemcpyDeviceToHost, s));
    return SOBEL5_OK;
}

void finish_staged(sobel5_ctx* ctx, void* const staged[7], int out_w, int rows) {
    for (int i = 0; i < 7; ++i)
        if (staged[i])
            par_copy(ctx, staged[i], ctx->h_stage[i], static_cast<size_t>(out_w) * kElem[i] * rows);
}

// Enqueues the chunked H2D -> kernel -> D2H pipeline of run_stream on the
// context's streams.  dst[i] is the host destination of plane i (tightly
// packed, out_w pitch), or nullptr with bit i of `mask` set to land the
// plane in the pinned staging buffer h_stage[i].  ev_out[k] marks chunk k's
// downloads.
// (op = 5: the 4-direction 5x5 operator, sobel5_launch; op = 3: the 3x3
// two-direction one, sobel3_launch, taps unused.)
sobel5_status enqueue_stream(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                             const sobel5_taps* taps, int prefetch, unsigned mask,
                             void* const dst[7], int* chunk_out, int* n_chunks_out,
                             StageBudget& budget, int op = 5, bool wire = false,
                             bool chunk_major = false, bool host_g = false) {
    const int R = op == 3 ? 1 : 2;  // operator radius
    ctx->wire = wire;
    ctx->wire_cm = wire && chunk_major;
    ctx->wire_g = ctx->wire_cm && host_g && ((mask >> 4) & 1u);
    ctx->wire_np = op == 3 ? 2 : 4;
    const int np = ctx->wire_np;
    const int out_w = width - 2 * R, out_h = height - 2 * R;
    const int64_t in_pitch = round_up(width, 128);
    const int64_t dpitch = round_up(out_w, 32);  // elements; 128 B-aligned int rows
    CK(ensure(reinterpret_cast<void**>(&ctx->d_in), &ctx->d_in_bytes,
              static_cast<size_t>(in_pitch) * height));
    const uint8_t* src_in = nullptr;
    if (const sobel5_status st =
            stage_input(ctx, h_in, static_cast<size_t>(width) * height, &src_in, budget);
        st != SOBEL5_OK)
        return st;
    sobel5_planes dp{};
    dp.pitch = dpitch;
    void** dslots[7] = {reinterpret_cast<void**>(&dp.gx),  reinterpret_cast<void**>(&dp.gy),
                        reinterpret_cast<void**>(&dp.gd),  reinterpret_cast<void**>(&dp.gdt),
                        reinterpret_cast<void**>(&dp.g),   reinterpret_cast<void**>(&dp.g32),
                        reinterpret_cast<void**>(&dp.u8)};
    void* hdst[7] = {};
    for (int i = 0; i < 7; ++i) {
        if (!((mask >> i) & 1u) || (i == 4 && ctx->wire_g)) continue;
        const size_t plane_bytes = static_cast<size_t>(out_w) * out_h * wire_elem(ctx, i);
        if (ctx->wire_cm && i < np) {
            // block of the np int16 planes, padded rows (dpitch); the
            // per-chunk plane pointers are set at the launches
            const size_t wb = np * static_cast<size_t>(dpitch) * out_h * 2;
            CK(ensure(&ctx->d_wire, &ctx->d_wire_bytes, wb));
            CK(ensure_host(&ctx->h_wire[0], &ctx->h_wire_bytes[0], wb));
            *dslots[i] = ctx->d_wire;
            hdst[i] = ctx->h_wire[0];
            continue;
        }
        CK(ensure(&ctx->d_plane[i], &ctx->d_plane_bytes[i],
                  static_cast<size_t>(dpitch) * out_h * kElem[i]));
        *dslots[i] = ctx->d_plane[i];
        if (wire && i < np) {
            CK(ensure_host(&ctx->h_wire[i], &ctx->h_wire_bytes[i], plane_bytes));
            hdst[i] = ctx->h_wire[i];
        } else if (dst[i]) {
            hdst[i] = dst[i];
        } else {
            CK(ensure_host(&ctx->h_stage[i], &ctx->h_stage_bytes[i], plane_bytes));
            hdst[i] = ctx->h_stage[i];
        }
    }

    // Row chunks: enough to overlap copies with compute, few enough that
    // each kernel still fills the GPU.
    // (16 for sobel5_run_host's int16 wire: the host widening of chunk k
    // overlaps the download of chunk k+1, so shorter chunks expose less of
    // it; the split form's consumers synchronise per chunk and prefer 8)
    const char* cv = std::getenv("SOBEL5_CHUNKS");
    const int n_want = cv && *cv && std::atoi(cv) > 0 ? std::atoi(cv) : (ctx->wire_cm ? 16 : 8);
    int chunk = std::max(256, (out_h + n_want - 1) / n_want);
    chunk = std::min(chunk, out_h);
    const int n_chunks = (out_h + chunk - 1) / chunk;
    ctx->wire_pitch = dpitch;
    CK(ensure_events(ctx->ev_in, static_cast<size_t>(n_chunks)));
    CK(ensure_events(ctx->ev_comp, static_cast<size_t>(n_chunks)));
    CK(ensure_events(ctx->ev_out, static_cast<size_t>(n_chunks)));
    CK(reset_diag(ctx));

    ctx->last_d2h = 0;
    int uploaded = 0;  // input rows already enqueued
    for (int k = 0; k < n_chunks; ++k) {
        const int y0 = k * chunk, y1 = std::min(out_h, y0 + chunk);
        const int need = y1 + 2 * R;  // input rows [y0, y1 + 2R)
        CK(cudaMemcpy2DAsync(ctx->d_in + static_cast<int64_t>(uploaded) * in_pitch, in_pitch,
                             src_in + static_cast<int64_t>(uploaded) * width, width, width,
                             need - uploaded, cudaMemcpyHostToDevice, ctx->s_h2d));
        uploaded = need;
        CK(cudaEventRecord(ctx->ev_in[k], ctx->s_h2d));
        CK(cudaStreamWaitEvent(ctx->s_comp, ctx->ev_in[k], 0));
        sobel5_planes sub = dp;
        const int64_t off = static_cast<int64_t>(y0) * dpitch;
        // int16 wire planes: the kernel addresses them as int16 at the int32
        // pointer (dpitch is even, so the chunk starts on an int32 boundary)
        const int64_t off_g = wire ? off / 2 : off;
        if (ctx->wire_cm) {
            // chunk k's block: plane p at (4 k chunk + p (y1 - y0)) rows
            int16_t* blk = static_cast<int16_t*>(ctx->d_wire) + np * static_cast<int64_t>(y0) * dpitch;
            const int64_t ps = static_cast<int64_t>(y1 - y0) * dpitch;
            sub.gx = reinterpret_cast<int32_t*>(blk);
            sub.gy = reinterpret_cast<int32_t*>(blk + ps);
            if (np == 4) {
                sub.gd = reinterpret_cast<int32_t*>(blk + 2 * ps);
                sub.gdt = reinterpret_cast<int32_t*>(blk + 3 * ps);
            }
        } else {
            if (sub.gx) sub.gx += off_g;
            if (sub.gy) sub.gy += off_g;
            if (sub.gd) sub.gd += off_g;
            if (sub.gdt) sub.gdt += off_g;
        }
        if (sub.g) sub.g += off;
        if (sub.g32) sub.g32 += off;
        if (sub.u8) sub.u8 += off;
        const uint8_t* d_rows = ctx->d_in + static_cast<int64_t>(y0) * in_pitch;
        sobel5_b200::LaunchExtra ex;
        ex.n16 = wire ? 1 : 0;
        ex.row0 = y0;  // the chunk's rows in the image: a global ParityViolation key
        const sobel5_status st =
            op == 3 ? sobel5_b200::sobel3_common(d_rows, in_pitch, 0, width, y1 - y0 + 2, 1, prefetch,
                                                 &sub, 0, ctx->s_comp, ex)
                    : sobel5_b200::launch_common(nullptr, d_rows, nullptr, in_pitch, 0, width,
                                                 y1 - y0 + 4, 1, taps, prefetch, &sub, 0,
                                                 ctx->d_diag, ctx->s_comp, ex);
        if (st != SOBEL5_OK) {
            ctx->last_error = cudaGetErrorString(cudaGetLastError());
            return st;
        }
        CK(cudaEventRecord(ctx->ev_comp[k], ctx->s_comp));
        CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_comp[k], 0));
        if (ctx->wire_cm) {  // the four int16 planes of the chunk: one copy
            const size_t off = np * static_cast<size_t>(y0) * dpitch * 2;
            const size_t n = np * static_cast<size_t>(y1 - y0) * dpitch * 2;
            ctx->last_d2h += n;
            CK(cudaMemcpyAsync(static_cast<char*>(ctx->h_wire[0]) + off,
                               static_cast<const char*>(ctx->d_wire) + off, n,
                               cudaMemcpyDeviceToHost, ctx->s_d2h));
        }
        for (int i = 0; i < 7; ++i) {
            if (!hdst[i] || (ctx->wire_cm && i < np)) continue;
            const size_t es = wire_elem(ctx, i);
            ctx->last_d2h += static_cast<uint64_t>(out_w) * es * static_cast<uint64_t>(y1 - y0);
            CK(cudaMemcpy2DAsync(static_cast<char*>(hdst[i]) + static_cast<size_t>(y0) * out_w * es,
                                 static_cast<size_t>(out_w) * es,
                                 static_cast<char*>(ctx->d_plane[i]) +
                                     static_cast<size_t>(y0) * dpitch * es,
                                 static_cast<size_t>(dpitch) * es, static_cast<size_t>(out_w) * es,
                                 static_cast<size_t>(y1 - y0), cudaMemcpyDeviceToHost,
                                 ctx->s_d2h));
        }
        CK(cudaEventRecord(ctx->ev_out[k], ctx->s_d2h));
    }
    CK(cudaMemcpyAsync(ctx->h_diag, ctx->d_diag, sizeof(sobel5_diag), cudaMemcpyDeviceToHost,
                       ctx->s_d2h));
    *chunk_out = chunk;
    *n_chunks_out = n_chunks;
    return SOBEL5_OK;
}

// Waits for the downloads chunk by chunk and moves the staged planes
// (stage_dst[i] != nullptr) into the caller's pageable memory while the later
// chunks are still in flight: every staged plane's rows of the chunk are cut
// into ~1 MiB pieces copied by the whole pool at once.
sobel5_status drain_stream(sobel5_ctx* ctx, int out_w, int out_h, int chunk, int n_chunks,
                           void* const stage_dst[7], sobel5_diag* diag_out) {
    constexpr size_t kPiece = size_t{1} << 20;
    struct Piece {
        char* dst;
        const char* src;
        size_t n;     // bytes of src (rows: row count)
        bool widen;   // int16 wire -> int32 destination
        bool rows = false;  // chunk-major wire: n rows of out_w, source pitch wire_pitch
    };
    std::vector<Piece> pieces;
    for (int k = 0; k < n_chunks; ++k) {
        CK(cudaEventSynchronize(ctx->ev_out[k]));
        const int y0 = k * chunk, y1 = std::min(out_h, y0 + chunk);
        pieces.clear();
        if (ctx->wire_g) {
            // rows of the chunk's int16 planes widened + g rebuilt, ~1 MiB of
            // output per piece
            const int64_t dp = ctx->wire_pitch, rows = y1 - y0;
            const int np = ctx->wire_np;
            const int per = decode_rows_per_piece(ctx, static_cast<int>(rows), out_w);
            const int n_pieces = static_cast<int>((rows + per - 1) / per);
            const int16_t* blk = static_cast<const int16_t*>(ctx->h_wire[0]) + np * static_cast<int64_t>(y0) * dp;
            void* dst[7] = {};
            for (int i = 0; i < 7; ++i)
                if (stage_dst[i] && (i < np || i == 4))
                    dst[i] = static_cast<char*>(stage_dst[i]) +
                             static_cast<size_t>(y0) * out_w * kElem[i];
            auto dec = [&](int t) {
                const int64_t r0 = static_cast<int64_t>(t) * per;
                decode_wire_rows(dst, blk, np, rows, dp, out_w, r0, std::min<int64_t>(per, rows - r0),
                                 dst[4] != nullptr);
            };
            if (n_pieces == 1) dec(0);
            else ctx->pool.run(n_pieces, dec);
        } else if (ctx->wire_cm) {
            // rows of the chunk's four int16 planes, ~1 MiB of output per piece
            const int64_t dp = ctx->wire_pitch, rows = y1 - y0;
            const int per = std::max<int64_t>(1, (int64_t{1} << 18) / std::max(out_w, 1));
            const int np = ctx->wire_np;
            const int16_t* blk = static_cast<const int16_t*>(ctx->h_wire[0]) + np * static_cast<int64_t>(y0) * dp;
            for (int i = 0; i < np; ++i) {
                if (!stage_dst[i]) continue;
                for (int64_t r = 0; r < rows; r += per)
                    pieces.push_back({static_cast<char*>(stage_dst[i]) +
                                          (static_cast<size_t>(y0 + r) * out_w) * 4,
                                      reinterpret_cast<const char*>(blk + (i * rows + r) * dp),
                                      static_cast<size_t>(std::min<int64_t>(per, rows - r)), true, true});
            }
        }
        for (int i = 0; i < 7; ++i) {
            if (!stage_dst[i] || (ctx->wire_cm && i < ctx->wire_np) || (i == 4 && ctx->wire_g))
                continue;
            const bool widen = ctx->wire && i < ctx->wire_np;
            const size_t es = wire_elem(ctx, i), row = static_cast<size_t>(out_w) * es;
            const size_t off = static_cast<size_t>(y0) * row, n = static_cast<size_t>(y1 - y0) * row;
            const char* src = static_cast<const char*>(widen ? ctx->h_wire[i] : ctx->h_stage[i]);
            for (size_t o = 0; o < n; o += kPiece)
                pieces.push_back({static_cast<char*>(stage_dst[i]) + (widen ? 2 : 1) * (off + o),
                                  src + off + o, std::min(kPiece, n - o), widen, false});
        }
        auto move = [&](const Piece& q) {
            if (q.rows) {
                for (size_t r = 0; r < q.n; ++r)
                    sobel5_b200::widen_i16(reinterpret_cast<int32_t*>(q.dst) + r * out_w,
                                           reinterpret_cast<const int16_t*>(q.src) + r * ctx->wire_pitch,
                                           static_cast<size_t>(out_w));
            } else if (q.widen)
                sobel5_b200::widen_i16(reinterpret_cast<int32_t*>(q.dst),
                                       reinterpret_cast<const int16_t*>(q.src), q.n / 2);
            else
                std::memcpy(q.dst, q.src, q.n);
        };
        if (pieces.size() == 1) {
            move(pieces[0]);
        } else if (!pieces.empty()) {
            ctx->pool.run(static_cast<int>(pieces.size()), [&](int t) { move(pieces[t]); });
        }
    }
    CK(cudaStreamSynchronize(ctx->s_d2h));
    if (diag_out) *diag_out = *ctx->h_diag;
    return ctx->h_diag->violations ? SOBEL5_PARITY_VIOLATION : SOBEL5_OK;
}

void planes_array(const sobel5_planes* p, void* out[7]) {
    out[0] = p->gx; out[1] = p->gy; out[2] = p->gd; out[3] = p->gdt;
    out[4] = p->g; out[5] = p->g32; out[6] = p->u8;
}

}  // namespace

extern "C" {

sobel5_status sobel5_ctx_create(sobel5_ctx** out, int device) {
    if (!out) return SOBEL5_INVALID_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return SOBEL5_NO_DEVICE;
    if (device < 0 || device >= n) return SOBEL5_INVALID_ARG;
    auto* ctx = new sobel5_ctx;
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->s_comp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->d_diag, sizeof(sobel5_diag));
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_diag, 2 * sizeof(sobel5_diag));
    if (e != cudaSuccess) {
        sobel5_ctx_destroy(ctx);
        return e == cudaErrorMemoryAllocation ? SOBEL5_OUT_OF_MEMORY : SOBEL5_CUDA_ERROR;
    }
    *out = ctx;
    return SOBEL5_OK;
}

void sobel5_ctx_destroy(sobel5_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (auto s : {ctx->s_h2d, ctx->s_comp, ctx->s_d2h})
        if (s) cudaStreamSynchronize(s);
    for (auto ev : ctx->ev_in) cudaEventDestroy(ev);
    for (auto ev : ctx->ev_comp) cudaEventDestroy(ev);
    for (auto ev : ctx->ev_out) cudaEventDestroy(ev);
    if (ctx->d_in) cudaFree(ctx->d_in);
    if (ctx->d_wire) cudaFree(ctx->d_wire);
    if (ctx->f_d_in) cudaFree(ctx->f_d_in);
    if (ctx->f_d_out) cudaFree(ctx->f_d_out);
    if (ctx->f_h_stage) cudaFreeHost(ctx->f_h_stage);
    for (auto ev : ctx->f_ev) cudaEventDestroy(ev);
    for (void* p : ctx->d_plane)
        if (p) cudaFree(p);
    for (void* p : ctx->h_stage)
        if (p) cudaFreeHost(p);
    for (void* p : ctx->h_wire)
        if (p) cudaFreeHost(p);
    if (ctx->h_in_stage) cudaFreeHost(ctx->h_in_stage);
    if (ctx->d_diag) cudaFree(ctx->d_diag);
    if (ctx->d_scratch) cudaFree(ctx->d_scratch);
    if (ctx->h_diag) cudaFreeHost(ctx->h_diag);
    for (auto s : {ctx->s_h2d, ctx->s_comp, ctx->s_d2h})
        if (s) cudaStreamDestroy(s);
    delete ctx;
}

uint64_t sobel5_ctx_last_d2h_bytes(const sobel5_ctx* ctx) { return ctx ? ctx->last_d2h : 0; }

sobel5_status sobel5_ctx_set_strip_width(sobel5_ctx* ctx, int strip_w) {
    if (!ctx || strip_w < 0) return SOBEL5_INVALID_ARG;
    ctx->strip_w = strip_w;
    return SOBEL5_OK;
}

const char* sobel5_ctx_last_error(const sobel5_ctx* ctx) {
    return ctx ? ctx->last_error.c_str() : "";
}

sobel5_status sobel5_run_host(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                              const sobel5_taps* taps, int prefetch, const sobel5_planes* h_out,
                              sobel5_diag* diag_out) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    // pipeline.hpp:454-456 first
    if (width < 5 || height < 5) return SOBEL5_IMAGE_TOO_SMALL;
    if (!h_in || !taps || !h_out) return SOBEL5_INVALID_ARG;
    if (ctx->pend.active) return SOBEL5_INVALID_ARG;  // a begin() awaits its finish()
    const int out_w = width - 4, out_h = height - 4;
    if (h_out->pitch != out_w) return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    void* hp[7];
    planes_array(h_out, hp);
    unsigned mask = 0;
    for (int i = 0; i < 7; ++i)
        if (hp[i]) mask |= 1u << i;
    // The StreamResult over the int16 wire with g rebuilt on the host runs
    // as a one-frame stream: row chunks through a small ring of device and
    // pinned staging slots, the decode of chunk k overlapping the downloads
    // of the next ones (8K: 8.1-8.3 vs 8.9-9.1 ms for the whole-image
    // staging, profiles/r2/frames_ring2.txt).  SOBEL5_RUN_HOST_RING=0 keeps
    // the whole-image form.
    if (want_wire(mask, taps, 5, false) && want_host_g() &&
        !(std::getenv("SOBEL5_RUN_HOST_RING") && std::atoi(std::getenv("SOBEL5_RUN_HOST_RING")) == 0))
        return sobel5_run_host_frames(ctx, h_in, width, height, 1, static_cast<int64_t>(width) * height,
                                      taps, prefetch, h_out, static_cast<int64_t>(out_w) * out_h,
                                      diag_out);
    void* direct[7] = {};  // pinned destinations: DMA straight into them
    void* staged[7] = {};  // pageable ones: through pinned staging (and the int16 wire planes)
    StageBudget budget;    // the planes first, then the input if it still fits
    const size_t n_px = static_cast<size_t>(out_w) * out_h;
    const bool wire = want_wire(mask, taps, 5, false) &&
                      budget.take(4 * static_cast<size_t>(round_up(out_w, 32)) * out_h * 2);
    const bool host_g = wire && want_host_g();
    for (int i = 0; i < 7; ++i) {
        if (!hp[i]) continue;
        if (wire && (i < 4 || (i == 4 && host_g))) {
            staged[i] = hp[i];  // widened (g: rebuilt) from the int16 staging
            continue;
        }
        if (!is_pinned(hp[i]) && budget.take(n_px * kElem[i]))
            staged[i] = hp[i];
        else
            direct[i] = hp[i];  // pinned, or over the staging cap: driver-staged copy
    }
    int chunk = 0, n_chunks = 0;
    const sobel5_status st = enqueue_stream(ctx, h_in, width, height, taps, prefetch, mask, direct,
                                            &chunk, &n_chunks, budget, 5, wire, true, host_g);
    if (st != SOBEL5_OK) return st;
    return drain_stream(ctx, out_w, out_h, chunk, n_chunks, staged, diag_out);
}

// Frames end to end (sobel5_run_host_frames): the units are row chunks of
// the frames (one per frame up to ~4 M output px, else the row chunks of
// sobel5_run_host), kept kFrameSlots in flight on the three streams through
// rings of kFrameSlots + 1 device input / output slots and pinned staging
// slots.  Once unit u's download has landed the host enqueues unit
// u + kFrameSlots -- into the slot of unit u - 1, already widened / copied
// out, so no device-side slot waits are needed -- and then decodes unit u
// while the device works on the next ones.  With default taps and the five
// StreamResult planes gx..gdt ride the int16 wire (chunk-major block per
// unit); other pinned destinations are DMA'd straight into, pageable ones go
// through the unit's staging slot.
sobel5_status sobel5_run_host_frames(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                                     int n_frames, int64_t in_frame_stride, const sobel5_taps* taps,
                                     int prefetch, const sobel5_planes* h_out,
                                     int64_t out_frame_stride, sobel5_diag* diag_out) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    if (width < 5 || height < 5) return SOBEL5_IMAGE_TOO_SMALL;  // pipeline.hpp:454-456
    if (!h_in || !taps || !h_out || n_frames < 1) return SOBEL5_INVALID_ARG;
    if (ctx->pend.active) return SOBEL5_INVALID_ARG;
    const int out_w = width - 4, out_h = height - 4;
    const int64_t out_px = static_cast<int64_t>(out_w) * out_h;
    if (h_out->pitch != out_w || in_frame_stride < static_cast<int64_t>(width) * height ||
        out_frame_stride < out_px)
        return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    // units in flight (SOBEL5_FRAME_SLOTS, 2..16) and row chunks per large
    // frame (SOBEL5_FRAME_CHUNKS): experiment knobs
    const char* sv = std::getenv("SOBEL5_FRAME_SLOTS");
    const int kFrameSlots = sv && *sv ? std::min(16, std::max(2, std::atoi(sv))) : 4;
    const int n_slots = kFrameSlots + 1;
    const char* cv = std::getenv("SOBEL5_FRAME_CHUNKS");
    const int frame_chunks = cv && *cv && std::atoi(cv) > 0 ? std::atoi(cv) : 32;
    void* hp[7];
    planes_array(h_out, hp);
    unsigned mask = 0;
    for (int i = 0; i < 7; ++i)
        if (hp[i]) mask |= 1u << i;
    if (!mask) return SOBEL5_OK;
    const bool wire = want_wire(mask, taps, 5, false);
    const bool host_g = wire && want_host_g();  // g rebuilt on the host from the wire
    ctx->wire = false;  // (the single-call wire state is not used here)
    const int64_t in_pitch = round_up(width, 128);
    const int64_t dpitch = round_up(out_w, 32);
    // units: whole frames up to ~4 M output px, else frame_chunks row chunks,
    // more when a unit's output would pass ~96 MB (the pinned staging of the
    // ring stays bounded for any image: 32K x 32K takes 128-row units)
    const int64_t row_out_bytes = static_cast<int64_t>(dpitch) * 24;
    const int cap_rows = static_cast<int>(std::max<int64_t>(64, (int64_t{96} << 20) / row_out_bytes));
    const int chunk = out_px <= (int64_t{4} << 20)
                          ? out_h
                          : std::min({out_h, cap_rows,
                                      std::max(64, (out_h + frame_chunks - 1) / frame_chunks)});
    const int n_chunks = (out_h + chunk - 1) / chunk;
    const int64_t n_units = static_cast<int64_t>(n_frames) * n_chunks;
    // slot layouts (bytes): device [input rows][wire block | planes], host
    // staging [wire block | pageable planes]
    const size_t in_slot = static_cast<size_t>(in_pitch) * (chunk + 4);
    size_t dev_off[7] = {}, host_off[7] = {}, dev_slot = 0, host_slot = 0;
    bool pinned[7] = {};
    const size_t wire_bytes = wire ? 4 * static_cast<size_t>(chunk) * dpitch * 2 : 0;
    dev_slot = host_slot = wire_bytes;
    for (int i = 0; i < 7; ++i) {
        if (!hp[i] || (wire && i < 4) || (host_g && i == 4)) continue;
        dev_off[i] = dev_slot;
        dev_slot += round_up(static_cast<int64_t>(chunk) * dpitch * kElem[i], 256);
        pinned[i] = is_pinned(hp[i]);
        if (!pinned[i]) {
            host_off[i] = host_slot;
            host_slot += round_up(static_cast<int64_t>(chunk) * out_w * kElem[i], 256);
        }
    }
    dev_slot = round_up(static_cast<int64_t>(dev_slot), 256);
    host_slot = round_up(static_cast<int64_t>(std::max<size_t>(host_slot, 256)), 256);
    CK(ensure(&ctx->f_d_in, &ctx->f_d_in_bytes, n_slots * in_slot));
    CK(ensure(&ctx->f_d_out, &ctx->f_d_out_bytes, n_slots * dev_slot));
    CK(ensure_host(&ctx->f_h_stage, &ctx->f_h_stage_bytes, n_slots * host_slot));
    CK(ensure_events(ctx->f_ev, 3 * n_slots));
    CK(reset_diag(ctx));
    const uint8_t* src_in = h_in;  // pageable input: the driver stages the (small) uploads
    ctx->last_d2h = 0;

    auto unit_rows = [&](int64_t u, int& f, int& y0, int& y1) {
        f = static_cast<int>(u / n_chunks);
        y0 = static_cast<int>(u % n_chunks) * chunk;
        y1 = std::min(out_h, y0 + chunk);
    };
    auto enqueue_unit = [&](int64_t u) -> sobel5_status {
        int f, y0, y1;
        unit_rows(u, f, y0, y1);
        const int slot = static_cast<int>(u % n_slots), rows = y1 - y0;
        cudaEvent_t ev_in = ctx->f_ev[3 * slot], ev_comp = ctx->f_ev[3 * slot + 1],
                    ev_out = ctx->f_ev[3 * slot + 2];
        uint8_t* d_in = static_cast<uint8_t*>(ctx->f_d_in) + slot * in_slot;
        char* d_out = static_cast<char*>(ctx->f_d_out) + slot * dev_slot;
        char* h_st = static_cast<char*>(ctx->f_h_stage) + slot * host_slot;
        // input rows [y0, y1 + 4) of frame f
        CK(cudaMemcpy2DAsync(d_in, in_pitch,
                             src_in + static_cast<int64_t>(f) * in_frame_stride +
                                 static_cast<int64_t>(y0) * width,
                             width, width, rows + 4, cudaMemcpyHostToDevice, ctx->s_h2d));
        CK(cudaEventRecord(ev_in, ctx->s_h2d));
        CK(cudaStreamWaitEvent(ctx->s_comp, ev_in, 0));
        sobel5_planes sub{};
        sub.pitch = dpitch;
        int32_t** islots[4] = {&sub.gx, &sub.gy, &sub.gd, &sub.gdt};
        for (int i = 0; i < 4; ++i) {
            if (!hp[i]) continue;
            *islots[i] = reinterpret_cast<int32_t*>(
                wire ? d_out + static_cast<size_t>(i) * rows * dpitch * 2 : d_out + dev_off[i]);
        }
        if (hp[4] && !host_g) sub.g = reinterpret_cast<double*>(d_out + dev_off[4]);
        if (hp[5]) sub.g32 = reinterpret_cast<float*>(d_out + dev_off[5]);
        if (hp[6]) sub.u8 = reinterpret_cast<uint8_t*>(d_out + dev_off[6]);
        sobel5_b200::LaunchExtra ex;
        ex.n16 = wire ? 1 : 0;
        ex.frame0 = f;  // the ParityViolation key: frame, then strip, row, column
        ex.row0 = y0;
        const sobel5_status st = sobel5_b200::launch_common(nullptr, d_in, nullptr, in_pitch, 0, width,
                                                            rows + 4, 1, taps, prefetch, &sub, 0,
                                                            ctx->d_diag, ctx->s_comp, ex);
        if (st != SOBEL5_OK) {
            ctx->last_error = cudaGetErrorString(cudaGetLastError());
            return st;
        }
        CK(cudaEventRecord(ev_comp, ctx->s_comp));
        CK(cudaStreamWaitEvent(ctx->s_d2h, ev_comp, 0));
        if (wire) {
            const size_t n = 4 * static_cast<size_t>(rows) * dpitch * 2;
            CK(cudaMemcpyAsync(h_st, d_out, n, cudaMemcpyDeviceToHost, ctx->s_d2h));
            ctx->last_d2h += n;
        }
        for (int i = 0; i < 7; ++i) {
            if (!hp[i] || (wire && i < 4) || (host_g && i == 4)) continue;
            const size_t es = kElem[i];
            void* dst = pinned[i] ? static_cast<char*>(hp[i]) +
                                        (static_cast<size_t>(f) * out_frame_stride +
                                         static_cast<size_t>(y0) * out_w) * es
                                  : h_st + host_off[i];
            CK(cudaMemcpy2DAsync(dst, static_cast<size_t>(out_w) * es, d_out + dev_off[i],
                                 static_cast<size_t>(dpitch) * es, static_cast<size_t>(out_w) * es,
                                 rows, cudaMemcpyDeviceToHost, ctx->s_d2h));
            ctx->last_d2h += static_cast<uint64_t>(rows) * out_w * es;
        }
        CK(cudaEventRecord(ev_out, ctx->s_d2h));
        return SOBEL5_OK;
    };
    // host side of unit u: wire planes widened, staged planes copied out
    struct Piece {
        int plane;  // -1: the wire planes + g rebuilt, from row `rows` on
        const char* src;
        char* dst;
        int rows;
    };
    std::vector<Piece> pieces;
    auto finish_unit = [&](int64_t u) {
        int f, y0, y1;
        unit_rows(u, f, y0, y1);
        const int slot = static_cast<int>(u % n_slots), rows = y1 - y0;
        const char* h_st = static_cast<const char*>(ctx->f_h_stage) + slot * host_slot;
        const int per = std::max(1, (1 << 18) / std::max(out_w, 1));
        pieces.clear();
        // gx..gdt widened and g rebuilt together: the unit's rows split evenly
        // over the pool (one wave; 1 MiB pieces left up to 40% of the threads
        // idle in the second wave of a 1/32 8K chunk)
        const int per_g = decode_rows_per_piece(ctx, rows, out_w);
        if (host_g)
            for (int r = 0; r < rows; r += per_g) pieces.push_back({-1, nullptr, nullptr, r});
        for (int i = 0; i < 7; ++i) {
            if (!hp[i] || (host_g && i <= 4)) continue;
            const bool w16 = wire && i < 4;
            if (!w16 && pinned[i]) continue;
            const size_t es = kElem[i];
            char* dst = static_cast<char*>(hp[i]) +
                        (static_cast<size_t>(f) * out_frame_stride + static_cast<size_t>(y0) * out_w) * es;
            const char* src = w16 ? h_st + static_cast<size_t>(i) * rows * dpitch * 2 : h_st + host_off[i];
            const size_t src_row = w16 ? static_cast<size_t>(dpitch) * 2 : static_cast<size_t>(out_w) * es;
            for (int r = 0; r < rows; r += per)
                pieces.push_back({i, src + r * src_row, dst + static_cast<size_t>(r) * out_w * es,
                                  std::min(per, rows - r)});
        }
        auto move = [&](const Piece& q) {
            const bool w16 = wire && q.plane < 4;
            if (q.plane < 0) {
                void* dst[7] = {};
                for (int i = 0; i < 5; ++i)
                    dst[i] = static_cast<char*>(hp[i]) +
                             (static_cast<size_t>(f) * out_frame_stride + static_cast<size_t>(y0) * out_w) *
                                 kElem[i];
                decode_wire_rows(dst, reinterpret_cast<const int16_t*>(h_st), 4, rows, dpitch, out_w,
                                 q.rows, std::min(per_g, rows - q.rows), true);
            } else if (w16) {
                for (int r = 0; r < q.rows; ++r)
                    sobel5_b200::widen_i16(reinterpret_cast<int32_t*>(q.dst) + static_cast<size_t>(r) * out_w,
                                           reinterpret_cast<const int16_t*>(q.src) + static_cast<size_t>(r) * dpitch,
                                           static_cast<size_t>(out_w));
            } else {
                std::memcpy(q.dst, q.src, static_cast<size_t>(q.rows) * out_w * kElem[q.plane]);
            }
        };
        if (pieces.size() == 1) move(pieces[0]);
        else if (!pieces.empty())
            ctx->pool.run(static_cast<int>(pieces.size()), [&](int t) { move(pieces[t]); });
    };
    sobel5_status st = SOBEL5_OK;
    for (int64_t u = 0; u < std::min<int64_t>(kFrameSlots, n_units) && st == SOBEL5_OK; ++u)
        st = enqueue_unit(u);
    cudaError_t wait_err = cudaSuccess;
    for (int64_t u = 0; u < n_units && st == SOBEL5_OK; ++u) {
        wait_err = cudaEventSynchronize(ctx->f_ev[3 * (u % n_slots) + 2]);
        if (wait_err != cudaSuccess) break;
        if (u + kFrameSlots < n_units) st = enqueue_unit(u + kFrameSlots);  // slot of unit u - 1
        finish_unit(u);
    }
    if (wait_err != cudaSuccess) return fail(ctx, wait_err);
    CK(cudaMemcpyAsync(ctx->h_diag, ctx->d_diag, sizeof(sobel5_diag), cudaMemcpyDeviceToHost,
                       ctx->s_d2h));
    CK(cudaStreamSynchronize(ctx->s_d2h));
    CK(cudaStreamSynchronize(ctx->s_comp));
    if (st != SOBEL5_OK) return st;
    if (diag_out) *diag_out = *ctx->h_diag;
    return ctx->h_diag->violations ? SOBEL5_PARITY_VIOLATION : SOBEL5_OK;
}

void sobel5_ctx_trim(sobel5_ctx* ctx) {
    if (!ctx || ctx->pend.active) return;
    cudaSetDevice(ctx->device);
    for (auto s : {ctx->s_h2d, ctx->s_comp, ctx->s_d2h}) cudaStreamSynchronize(s);
    for (int i = 0; i < 7; ++i) {
        if (ctx->h_stage[i]) cudaFreeHost(ctx->h_stage[i]);
        ctx->h_stage[i] = nullptr;
        ctx->h_stage_bytes[i] = 0;
        if (i < 4) {
            if (ctx->h_wire[i]) cudaFreeHost(ctx->h_wire[i]);
            ctx->h_wire[i] = nullptr;
            ctx->h_wire_bytes[i] = 0;
        }
        if (ctx->d_plane[i]) cudaFree(ctx->d_plane[i]);
        ctx->d_plane[i] = nullptr;
        ctx->d_plane_bytes[i] = 0;
    }
    if (ctx->h_in_stage) cudaFreeHost(ctx->h_in_stage);
    ctx->h_in_stage = nullptr;
    ctx->h_in_stage_bytes = 0;
    if (ctx->d_wire) cudaFree(ctx->d_wire);
    ctx->d_wire = nullptr;
    ctx->d_wire_bytes = 0;
    if (ctx->f_d_in) cudaFree(ctx->f_d_in);
    if (ctx->f_d_out) cudaFree(ctx->f_d_out);
    if (ctx->f_h_stage) cudaFreeHost(ctx->f_h_stage);
    ctx->f_d_in = ctx->f_d_out = ctx->f_h_stage = nullptr;
    ctx->f_d_in_bytes = ctx->f_d_out_bytes = ctx->f_h_stage_bytes = 0;
    if (ctx->d_in) cudaFree(ctx->d_in);
    ctx->d_in = nullptr;
    ctx->d_in_bytes = 0;
    if (ctx->d_scratch) cudaFree(ctx->d_scratch);
    ctx->d_scratch = nullptr;
    ctx->d_scratch_bytes = 0;
}

}  // extern "C"

namespace {
sobel5_status begin_common(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                           const sobel5_taps* taps, int prefetch, unsigned plane_mask, int op) {
    const int R = op == 3 ? 1 : 2;
    const bool wire = want_wire(plane_mask, taps, op, true);
    size_t stage_bytes = 0;
    for (int i = 0; i < 7; ++i)
        if ((plane_mask >> i) & 1u)
            stage_bytes += static_cast<size_t>(width - 2 * R) * (height - 2 * R) *
                           (wire && i < (op == 3 ? 2 : 4) ? 2 : kElem[i]);
    StageBudget budget;  // the planes must fit; the input is staged if it still does
    if (!budget.take(stage_bytes)) return SOBEL5_OUT_OF_MEMORY;  // callers use run_host
    CK(cudaSetDevice(ctx->device));
    void* none[7] = {};
    int chunk = 0, n_chunks = 0;
    const sobel5_status st = enqueue_stream(ctx, h_in, width, height, taps, prefetch, plane_mask,
                                            none, &chunk, &n_chunks, budget, op, wire);
    if (st != SOBEL5_OK) {
        // drain whatever was enqueued so the context stays usable
        cudaStreamSynchronize(ctx->s_h2d);
        cudaStreamSynchronize(ctx->s_comp);
        cudaStreamSynchronize(ctx->s_d2h);
        return st;
    }
    ctx->pend.active = true;
    ctx->pend.out_w = width - 2 * R;
    ctx->pend.out_h = height - 2 * R;
    ctx->pend.chunk = chunk;
    ctx->pend.n_chunks = n_chunks;
    ctx->pend.mask = plane_mask;
    return SOBEL5_OK;
}
}  // namespace

extern "C" {

sobel5_status sobel5_run_host_begin(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                                    const sobel5_taps* taps, int prefetch, unsigned plane_mask) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    if (width < 5 || height < 5) return SOBEL5_IMAGE_TOO_SMALL;
    if (!h_in || !taps || plane_mask == 0 || plane_mask >= (1u << 7) || ctx->pend.active)
        return SOBEL5_INVALID_ARG;
    return begin_common(ctx, h_in, width, height, taps, prefetch, plane_mask, 5);
}

sobel5_status sobel3_run_host_begin(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                                    int prefetch, unsigned plane_mask) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    if (width < 3 || height < 3) return SOBEL5_IMAGE_TOO_SMALL;  // pipeline.hpp:553-556
    // gd / gdt do not exist for the 3x3 operator
    if (!h_in || plane_mask == 0 || plane_mask >= (1u << 7) || (plane_mask & 0xcu) ||
        ctx->pend.active)
        return SOBEL5_INVALID_ARG;
    return begin_common(ctx, h_in, width, height, nullptr, prefetch, plane_mask, 3);
}

sobel5_status sobel5_run_host_finish(sobel5_ctx* ctx, const sobel5_planes* h_out,
                                     sobel5_diag* diag_out) {
    if (!ctx || !ctx->pend.active) return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    const auto pend = ctx->pend;
    void* hp[7] = {};
    bool ok = !h_out || h_out->pitch == pend.out_w;
    if (ok && h_out) {
        planes_array(h_out, hp);
        for (int i = 0; i < 7; ++i) ok = ok && ((hp[i] != nullptr) == (((pend.mask >> i) & 1u) != 0));
    }
    if (!ok) {  // still complete the pending work, then report the bad argument
        void* none[7] = {};
        drain_stream(ctx, pend.out_w, pend.out_h, pend.chunk, pend.n_chunks, none, nullptr);
        ctx->pend.active = false;
        return SOBEL5_INVALID_ARG;
    }
    const sobel5_status st =
        drain_stream(ctx, pend.out_w, pend.out_h, pend.chunk, pend.n_chunks, hp, diag_out);
    ctx->pend.active = false;
    return st;
}

sobel5_status sobel5_run_host_chunk(sobel5_ctx* ctx, int chunk, int* y0, int* y1) {
    if (!ctx || !ctx->pend.active || chunk < 0 || chunk >= ctx->pend.n_chunks || !y0 || !y1)
        return SOBEL5_INVALID_ARG;
    const cudaError_t e = cudaEventSynchronize(ctx->ev_out[chunk]);
    if (e != cudaSuccess) return SOBEL5_CUDA_ERROR;  // (last_error is not thread-safe)
    *y0 = chunk * ctx->pend.chunk;
    *y1 = std::min(ctx->pend.out_h, *y0 + ctx->pend.chunk);
    return SOBEL5_OK;
}

const void* sobel5_run_host_staging(const sobel5_ctx* ctx, int plane) {
    if (!ctx || !ctx->pend.active || plane < 0 || plane >= 7 || !((ctx->pend.mask >> plane) & 1u))
        return nullptr;
    return ctx->wire && plane < 4 ? ctx->h_wire[plane] : ctx->h_stage[plane];
}

int sobel5_run_host_staging_elem(const sobel5_ctx* ctx, int plane) {
    if (!ctx || !ctx->pend.active || plane < 0 || plane >= 7 || !((ctx->pend.mask >> plane) & 1u))
        return 0;
    return static_cast<int>(wire_elem(ctx, plane));
}

sobel5_status sobel5_detect_host(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                                 const sobel5_taps* taps, int prefetch, int pad, int save_mode,
                                 uint8_t* h_u8, const sobel5_planes* h_planes,
                                 sobel5_diag* diag_out) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    if (pad) {
        if (width < 1 || height < 1) return SOBEL5_EMPTY_PLANE;  // image_io.hpp:280
    } else if (width < 5 || height < 5) {
        return SOBEL5_IMAGE_TOO_SMALL;
    }
    if (!h_in || !taps || !h_u8 || (save_mode != 0 && save_mode != 1)) return SOBEL5_INVALID_ARG;
    const int out_w = pad ? width : width - 4, out_h = pad ? height : height - 4;
    if (h_planes && h_planes->pitch != out_w) return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    const int64_t in_pitch = round_up(width, 128);
    const int64_t dpitch = round_up(out_w, 32);
    CK(ensure(reinterpret_cast<void**>(&ctx->d_in), &ctx->d_in_bytes,
              static_cast<size_t>(in_pitch) * height));
    sobel5_planes dp{};
    dp.pitch = dpitch;
    void* hp[7] = {};
    if (h_planes) {
        hp[0] = h_planes->gx; hp[1] = h_planes->gy; hp[2] = h_planes->gd; hp[3] = h_planes->gdt;
        hp[4] = h_planes->g; hp[5] = h_planes->g32;
    }
    hp[6] = h_u8;
    void** dslots[7] = {reinterpret_cast<void**>(&dp.gx),  reinterpret_cast<void**>(&dp.gy),
                        reinterpret_cast<void**>(&dp.gd),  reinterpret_cast<void**>(&dp.gdt),
                        reinterpret_cast<void**>(&dp.g),   reinterpret_cast<void**>(&dp.g32),
                        reinterpret_cast<void**>(&dp.u8)};
    for (int i = 0; i < 7; ++i) {
        if (!hp[i]) continue;
        CK(ensure(&ctx->d_plane[i], &ctx->d_plane_bytes[i],
                  static_cast<size_t>(dpitch) * out_h * kElem[i]));
        *dslots[i] = ctx->d_plane[i];
    }
    CK(ensure(&ctx->d_scratch, &ctx->d_scratch_bytes,
              sobel5_detect_scratch_bytes(out_h, dpitch, 0, 1)));
    CK(reset_diag(ctx));
    StageBudget budget;
    const uint8_t* src_in = nullptr;
    if (const sobel5_status st =
            stage_input(ctx, h_in, static_cast<size_t>(width) * height, &src_in, budget);
        st != SOBEL5_OK)
        return st;
    CK(cudaMemcpy2DAsync(ctx->d_in, in_pitch, src_in, width, width, height, cudaMemcpyHostToDevice,
                         ctx->s_comp));
    const sobel5_status st = sobel5_detect(ctx->d_in, in_pitch, 0, width, height, 1, taps,
                                           prefetch, pad, save_mode, &dp, 0, ctx->d_scratch,
                                           ctx->d_diag, ctx->s_comp);
    if (st != SOBEL5_OK) {
        ctx->last_error = cudaGetErrorString(cudaGetLastError());
        return st;
    }
    void* staged[7] = {};
    for (int i = 0; i < 7; ++i) {
        if (!hp[i]) continue;
        if (const sobel5_status ds = download_plane(ctx, i, hp[i], ctx->d_plane[i], out_w, out_h,
                                                    dpitch, ctx->s_comp, staged, budget);
            ds != SOBEL5_OK)
            return ds;
    }
    CK(cudaMemcpyAsync(ctx->h_diag, ctx->d_diag, sizeof(sobel5_diag), cudaMemcpyDeviceToHost,
                       ctx->s_comp));
    CK(cudaStreamSynchronize(ctx->s_comp));
    finish_staged(ctx, staged, out_w, out_h);
    if (diag_out) *diag_out = *ctx->h_diag;
    return ctx->h_diag->violations ? SOBEL5_PARITY_VIOLATION : SOBEL5_OK;
}

sobel5_status sobel3_run_host(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                              int prefetch, const sobel5_planes* h_out) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    if (width < 3 || height < 3) return SOBEL5_IMAGE_TOO_SMALL;  // pipeline.hpp:553-556
    if (!h_in || !h_out || h_out->gd || h_out->gdt) return SOBEL5_INVALID_ARG;
    if (ctx->pend.active) return SOBEL5_INVALID_ARG;
    const int out_w = width - 2, out_h = height - 2;
    if (h_out->pitch != out_w) return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    // the same chunked upload / kernel / download pipeline as sobel5_run_host
    void* hp[7];
    planes_array(h_out, hp);
    unsigned mask = 0;
    for (int i = 0; i < 7; ++i)
        if (hp[i]) mask |= 1u << i;
    void* direct[7] = {};
    void* staged[7] = {};
    StageBudget budget;
    // gx, gy over the int16 wire (chunk-major), widened into the caller's planes
    const bool wire = want_wire(mask, nullptr, 3, false) &&
                      budget.take(2 * static_cast<size_t>(round_up(out_w, 32)) * out_h * 2);
    const bool host_g = wire && want_host_g();
    for (int i = 0; i < 7; ++i) {
        if (!hp[i]) continue;
        if (wire && (i < 2 || (i == 4 && host_g))) {
            staged[i] = hp[i];
            continue;
        }
        if (!is_pinned(hp[i]) && budget.take(static_cast<size_t>(out_w) * out_h * kElem[i]))
            staged[i] = hp[i];
        else
            direct[i] = hp[i];
    }
    if (!mask) return SOBEL5_OK;
    int chunk = 0, n_chunks = 0;
    const sobel5_status st = enqueue_stream(ctx, h_in, width, height, nullptr, prefetch, mask,
                                            direct, &chunk, &n_chunks, budget, 3, wire, true, host_g);
    if (st != SOBEL5_OK) return st;
    return drain_stream(ctx, out_w, out_h, chunk, n_chunks, staged, nullptr);
}

sobel5_status sobel5_quantize_host(sobel5_ctx* ctx, const void* h_plane, int kind, int width,
                                   int height, int save_mode, uint8_t* h_u8) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    if (width < 1 || height < 1) return SOBEL5_EMPTY_PLANE;  // image_io.hpp:259/265
    if (!h_plane || !h_u8 || kind < 0 || kind > 2) return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    const size_t es = kind == 0 ? sizeof(double) : kind == 1 ? sizeof(int32_t) : 1;
    const size_t n = static_cast<size_t>(width) * height;
    // the plane goes through the g slot (8 B/elem covers both kinds), u8 through u8
    CK(ensure(&ctx->d_plane[4], &ctx->d_plane_bytes[4], n * 8));
    CK(ensure(&ctx->d_plane[6], &ctx->d_plane_bytes[6], n));
    CK(ensure(&ctx->d_scratch, &ctx->d_scratch_bytes, sobel5_detect_scratch_bytes(0, 0, 0, 1)));
    StageBudget budget;
    const uint8_t* src = nullptr;
    if (const sobel5_status ss =
            stage_input(ctx, static_cast<const uint8_t*>(h_plane), n * es, &src, budget);
        ss != SOBEL5_OK)
        return ss;
    CK(cudaMemcpyAsync(ctx->d_plane[4], src, n * es, cudaMemcpyHostToDevice, ctx->s_comp));
    const sobel5_status st =
        sobel5_quantize_plane(ctx->d_plane[4], kind, width, width, height, save_mode,
                              static_cast<uint8_t*>(ctx->d_plane[6]), width, ctx->d_scratch,
                              ctx->s_comp);
    if (st != SOBEL5_OK) return st;
    void* staged[7] = {};
    if (const sobel5_status ds = download_plane(ctx, 6, h_u8, ctx->d_plane[6], width, height, width,
                                                ctx->s_comp, staged, budget);
        ds != SOBEL5_OK)
        return ds;
    CK(cudaStreamSynchronize(ctx->s_comp));
    finish_staged(ctx, staged, width, height);
    return SOBEL5_OK;
}

sobel5_status sobel5_conv2d_valid_host(sobel5_ctx* ctx, const uint8_t* h_in, int width,
                                       int height, const int32_t* kernel, int ksize,
                                       int32_t* h_out) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    if (ksize != 3 && ksize != 5) return SOBEL5_INVALID_ARG;
    if (width < ksize || height < ksize) return SOBEL5_IMAGE_TOO_SMALL;  // oracle.hpp:20-22
    if (!h_in || !kernel || !h_out || ctx->pend.active) return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    const int out_w = width - ksize + 1, out_h = height - ksize + 1;
    const int64_t in_pitch = round_up(width, 128);
    CK(ensure(reinterpret_cast<void**>(&ctx->d_in), &ctx->d_in_bytes,
              static_cast<size_t>(in_pitch) * height));
    // the int32 result goes through the gx slot, tightly packed
    CK(ensure(&ctx->d_plane[0], &ctx->d_plane_bytes[0], static_cast<size_t>(out_w) * out_h * 4));
    StageBudget budget;
    const uint8_t* src_in = nullptr;
    if (const sobel5_status st =
            stage_input(ctx, h_in, static_cast<size_t>(width) * height, &src_in, budget);
        st != SOBEL5_OK)
        return st;
    CK(cudaMemcpy2DAsync(ctx->d_in, in_pitch, src_in, width, width, height, cudaMemcpyHostToDevice,
                         ctx->s_comp));
    const sobel5_status st =
        sobel5_conv2d_valid(ctx->d_in, in_pitch, width, height, kernel, ksize,
                            static_cast<int32_t*>(ctx->d_plane[0]), out_w, ctx->s_comp);
    if (st != SOBEL5_OK) return st;
    void* staged[7] = {};
    if (const sobel5_status ds = download_plane(ctx, 0, h_out, ctx->d_plane[0], out_w, out_h,
                                                out_w, ctx->s_comp, staged, budget);
        ds != SOBEL5_OK)
        return ds;
    CK(cudaStreamSynchronize(ctx->s_comp));
    finish_staged(ctx, staged, out_w, out_h);
    return SOBEL5_OK;
}

sobel5_status sobel5_dense_4d_host(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                                   const int32_t* kernels, const sobel5_planes* h_out) {
    if (!ctx) return SOBEL5_INVALID_ARG;
    if (width < 5 || height < 5) return SOBEL5_IMAGE_TOO_SMALL;  // oracle.hpp:20-22
    if (!h_in || !kernels || !h_out || h_out->g32 || h_out->u8 || ctx->pend.active)
        return SOBEL5_INVALID_ARG;
    const int out_w = width - 4, out_h = height - 4;
    if (h_out->pitch != out_w) return SOBEL5_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    const int64_t in_pitch = round_up(width, 128);
    CK(ensure(reinterpret_cast<void**>(&ctx->d_in), &ctx->d_in_bytes,
              static_cast<size_t>(in_pitch) * height));
    void* hp[7];
    planes_array(h_out, hp);
    sobel5_planes dp{};
    dp.pitch = out_w;  // tightly packed device planes
    void** dslots[5] = {reinterpret_cast<void**>(&dp.gx), reinterpret_cast<void**>(&dp.gy),
                        reinterpret_cast<void**>(&dp.gd), reinterpret_cast<void**>(&dp.gdt),
                        reinterpret_cast<void**>(&dp.g)};
    for (int i = 0; i < 5; ++i) {
        if (!hp[i]) continue;
        CK(ensure(&ctx->d_plane[i], &ctx->d_plane_bytes[i],
                  static_cast<size_t>(out_w) * out_h * kElem[i]));
        *dslots[i] = ctx->d_plane[i];
    }
    StageBudget budget;
    const uint8_t* src_in = nullptr;
    if (const sobel5_status st =
            stage_input(ctx, h_in, static_cast<size_t>(width) * height, &src_in, budget);
        st != SOBEL5_OK)
        return st;
    CK(cudaMemcpy2DAsync(ctx->d_in, in_pitch, src_in, width, width, height, cudaMemcpyHostToDevice,
                         ctx->s_comp));
    const sobel5_status st = sobel5_dense_4d(ctx->d_in, in_pitch, width, height, kernels, &dp,
                                             ctx->s_comp);
    if (st != SOBEL5_OK) return st;
    void* staged[7] = {};
    for (int i = 0; i < 5; ++i) {
        if (!hp[i]) continue;
        if (const sobel5_status ds = download_plane(ctx, i, hp[i], ctx->d_plane[i], out_w, out_h,
                                                    out_w, ctx->s_comp, staged, budget);
            ds != SOBEL5_OK)
            return ds;
    }
    CK(cudaStreamSynchronize(ctx->s_comp));
    finish_staged(ctx, staged, out_w, out_h);
    return SOBEL5_OK;
}

}  // extern "C"
