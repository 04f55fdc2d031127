// wire_probe.cu -- is a narrow D2H wire format worth it for sobel5_run_host?
//
// The 8K StreamResult is 795 MB of int32/f64 planes; PCIe D2H (~55 GB/s)
// bounds the host call at ~14.5 ms.  With default taps every gradient fits
// int16, so the device could ship 4 x int16 + f64 = 16 B/px (530 MB) and the
// host widen the four gradient planes into the caller's int32 planes while
// later chunks are still on the wire.  This probe measures:
//   (1) D2H of 795 MB straight into pinned int32/f64 destinations (today)
//   (2) host widening int16 -> int32 of 4 x 33.1 M px on T threads, alone
//   (3) the pipelined narrow path: 8 row chunks, chunk k's int16 planes and
//       f64 plane DMA'd (f64 straight to the destination), the host widening
//       chunk k-1 on T threads meanwhile.
// Build: nvcc -O3 -std=c++17 -Xcompiler -mavx2,-pthread tools/probes/wire_probe.cu -o /tmp/wire_probe
#include <cuda_runtime.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t err_ = (x);                                                    \
        if (err_ != cudaSuccess) {                                               \
            std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(err_)); \
            std::exit(1);                                                       \
        }                                                                       \
    } while (0)

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// widen n int16 -> int32 with streaming stores (dst 32 B aligned pieces)
static void widen(int32_t* dst, const int16_t* src, size_t n, bool nt) {
    size_t i = 0;
    if (nt) {
        while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31)) { dst[i] = src[i]; ++i; }
        for (; i + 16 <= n; i += 16) {
            const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
            _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i),
                                _mm256_cvtepi16_epi32(_mm256_castsi256_si128(a)));
            _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 8),
                                _mm256_cvtepi16_epi32(_mm256_extracti128_si256(a, 1)));
        }
    } else {
        for (; i + 16 <= n; i += 16) {
            const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
            _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i),
                                _mm256_cvtepi16_epi32(_mm256_castsi256_si128(a)));
            _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i + 8),
                                _mm256_cvtepi16_epi32(_mm256_extracti128_si256(a, 1)));
        }
    }
    for (; i < n; ++i) dst[i] = src[i];
    _mm_sfence();
}

static void par(int T, size_t n, const std::function<void(size_t, size_t)>& f) {
    std::vector<std::thread> th;
    const size_t per = (n + T - 1) / T;
    for (int t = 0; t < T; ++t) {
        const size_t a = std::min(n, t * per), b = std::min(n, a + per);
        th.emplace_back([&, a, b] { f(a, b); });
    }
    for (auto& x : th) x.join();
}

int main() {
    const int W = 7676, H = 4316;
    const size_t N = static_cast<size_t>(W) * H;
    int16_t* d16[4];
    int32_t* d32[4];
    double* dg;
    for (int i = 0; i < 4; ++i) {
        CK(cudaMalloc(&d16[i], N * 2));
        CK(cudaMalloc(&d32[i], N * 4));
        CK(cudaMemset(d16[i], 1, N * 2));
    }
    CK(cudaMalloc(&dg, N * 8));
    int16_t* s16[4];
    int32_t* h32[4];
    double* hg;
    for (int i = 0; i < 4; ++i) {
        CK(cudaMallocHost(&s16[i], N * 2));
        CK(cudaMallocHost(&h32[i], N * 4));
        std::memset(s16[i], 1, N * 2);
        std::memset(h32[i], 0, N * 4);
    }
    CK(cudaMallocHost(&hg, N * 8));
    std::memset(hg, 0, N * 8);
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const unsigned hw = std::thread::hardware_concurrency();
    std::printf("hardware_concurrency %u, N %zu px\n", hw, N);

    // (1) today's D2H
    for (int rep = 0; rep < 3; ++rep) {
        const double t0 = now();
        for (int i = 0; i < 4; ++i) CK(cudaMemcpyAsync(h32[i], d32[i], N * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hg, dg, N * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const double dt = now() - t0;
        std::printf("(1) D2H int32x4 + f64 (795 MB): %.2f ms  %.1f GB/s\n", dt * 1e3, 24.0 * N / dt / 1e9);
    }
    for (int rep = 0; rep < 2; ++rep) {
        const double t0 = now();
        for (int i = 0; i < 4; ++i) CK(cudaMemcpyAsync(s16[i], d16[i], N * 2, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hg, dg, N * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const double dt = now() - t0;
        std::printf("    D2H int16x4 + f64 (530 MB): %.2f ms  %.1f GB/s\n", dt * 1e3, 16.0 * N / dt / 1e9);
    }
    // (2) widening alone
    for (int T : {1, 2, 4, 8, 12, 16}) {
        if (T > static_cast<int>(hw)) break;
        for (bool nt : {false, true}) {
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                const double t0 = now();
                par(T, 4 * N, [&](size_t a, size_t b) {
                    for (int i = 0; i < 4; ++i) {
                        const size_t lo = std::max(a, i * N), hi = std::min(b, (i + 1) * N);
                        if (lo < hi) widen(h32[i] + (lo - i * N), s16[i] + (lo - i * N), hi - lo, nt);
                    }
                });
                best = std::min(best, now() - t0);
            }
            std::printf("(2) widen 4 x %zu int16->int32, T=%2d %s: %.2f ms (%.1f GB/s written)\n", N, T,
                        nt ? "stream" : "store ", best * 1e3, 16.0 * N / best / 1e9);
        }
    }
    // (3) pipelined: 8 chunks; DMA chunk k while widening chunk k-1
    for (int T : {4, 8, 12, 16}) {
        if (T > static_cast<int>(hw)) break;
        for (int chunks : {8, 16, 32}) {
            std::vector<cudaEvent_t> ev(chunks);
            for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                const double t0 = now();
                const size_t rows = (H + chunks - 1) / chunks;
                for (int k = 0; k < chunks; ++k) {
                    const size_t o = std::min<size_t>(H, k * rows) * W, e = std::min<size_t>(H, (k + 1) * rows) * W;
                    for (int i = 0; i < 4; ++i)
                        CK(cudaMemcpyAsync(s16[i] + o, d16[i] + o, (e - o) * 2, cudaMemcpyDeviceToHost, s));
                    CK(cudaMemcpyAsync(hg + o, dg + o, (e - o) * 8, cudaMemcpyDeviceToHost, s));
                    CK(cudaEventRecord(ev[k], s));
                }
                for (int k = 0; k < chunks; ++k) {
                    CK(cudaEventSynchronize(ev[k]));
                    const size_t o = std::min<size_t>(H, k * rows) * W, e = std::min<size_t>(H, (k + 1) * rows) * W;
                    const size_t n = e - o;
                    par(T, 4 * n, [&](size_t a, size_t b) {
                        for (int i = 0; i < 4; ++i) {
                            const size_t lo = std::max(a, i * n), hi = std::min(b, (i + 1) * n);
                            if (lo < hi)
                                widen(h32[i] + o + (lo - i * n), s16[i] + o + (lo - i * n), hi - lo, true);
                        }
                    });
                }
                best = std::min(best, now() - t0);
            }
            std::printf("(3) narrow wire, %2d chunks, T=%2d: %.2f ms (= %.2f Gpx/s e2e-equivalent)\n", chunks, T,
                        best * 1e3, N / best / 1e9);
            for (auto& e : ev) cudaEventDestroy(e);
        }
    }
    // (4) k of the 4 gradient planes narrow (int16 + host widening), the
    // other 4-k int32 straight into the destination: 8 host threads, 16 chunks
    for (int k = 0; k <= 4; ++k) {
        const int chunks = 16, T = 8;
        std::vector<cudaEvent_t> ev(chunks);
        for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        double best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            const double t0 = now();
            const size_t rows = (H + chunks - 1) / chunks;
            for (int c = 0; c < chunks; ++c) {
                const size_t o = std::min<size_t>(H, c * rows) * W, e = std::min<size_t>(H, (c + 1) * rows) * W;
                for (int i = 0; i < 4; ++i) {
                    if (i < k) CK(cudaMemcpyAsync(s16[i] + o, d16[i] + o, (e - o) * 2, cudaMemcpyDeviceToHost, s));
                    else CK(cudaMemcpyAsync(h32[i] + o, d32[i] + o, (e - o) * 4, cudaMemcpyDeviceToHost, s));
                }
                CK(cudaMemcpyAsync(hg + o, dg + o, (e - o) * 8, cudaMemcpyDeviceToHost, s));
                CK(cudaEventRecord(ev[c], s));
            }
            for (int c = 0; c < chunks; ++c) {
                CK(cudaEventSynchronize(ev[c]));
                if (k == 0) continue;
                const size_t o = std::min<size_t>(H, c * rows) * W, e = std::min<size_t>(H, (c + 1) * rows) * W;
                const size_t n = e - o;
                par(T, static_cast<size_t>(k) * n, [&](size_t a, size_t b) {
                    for (int i = 0; i < k; ++i) {
                        const size_t lo = std::max(a, i * n), hi = std::min(b, (i + 1) * n);
                        if (lo < hi) widen(h32[i] + o + (lo - i * n), s16[i] + o + (lo - i * n), hi - lo, true);
                    }
                });
            }
            best = std::min(best, now() - t0);
        }
        std::printf("(4) %d of 4 gradient planes on the int16 wire: %.2f ms (%.2f Gpx/s)\n", k, best * 1e3,
                    N / best / 1e9);
        for (auto& e : ev) cudaEventDestroy(e);
    }
    // (5) chunk-major int16 blocks through a SMALL staging ring (slots
    // reused every `slots` chunks, so DMA writes may land in the host LLC
    // (DDIO) and the widening reads them from there): the D2H of chunk k is
    // enqueued once chunk k - slots has been widened
    for (int chunks : {16, 32, 64}) {
        for (int slots : {2, 3, 4, 8}) {
            const int T = 8;
            const size_t rows = (H + chunks - 1) / chunks;
            const size_t blk = 4 * rows * W;  // int16 elements per chunk block
            int16_t* ring = nullptr;
            CK(cudaMallocHost(&ring, blk * 2 * slots));
            int16_t* dblk = nullptr;
            CK(cudaMalloc(&dblk, blk * 2 * chunks));
            std::vector<cudaEvent_t> ev(chunks);
            for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                const double t0 = now();
                auto enqueue = [&](int c) {
                    const size_t y0 = std::min<size_t>(H, c * rows), y1 = std::min<size_t>(H, (c + 1) * rows);
                    const size_t n = 4 * (y1 - y0) * W;
                    CK(cudaMemcpyAsync(ring + (c % slots) * blk, dblk + c * blk, n * 2, cudaMemcpyDeviceToHost, s));
                    CK(cudaMemcpyAsync(hg + y0 * W, dg + y0 * W, (y1 - y0) * W * 8, cudaMemcpyDeviceToHost, s));
                    CK(cudaEventRecord(ev[c], s));
                };
                for (int c = 0; c < std::min(slots, chunks); ++c) enqueue(c);
                for (int c = 0; c < chunks; ++c) {
                    CK(cudaEventSynchronize(ev[c]));
                    const size_t y0 = std::min<size_t>(H, c * rows), y1 = std::min<size_t>(H, (c + 1) * rows);
                    const size_t n = (y1 - y0) * W;
                    const int16_t* src = ring + (c % slots) * blk;
                    par(T, 4 * n, [&](size_t a, size_t b) {
                        for (int i = 0; i < 4; ++i) {
                            const size_t lo = std::max(a, i * n), hi = std::min(b, (i + 1) * n);
                            if (lo < hi) widen(h32[i] + y0 * W + (lo - i * n), src + i * n + (lo - i * n), hi - lo, true);
                        }
                    });
                    if (c + slots < chunks) enqueue(c + slots);
                }
                best = std::min(best, now() - t0);
            }
            std::printf("(5) ring: %2d chunks, %d slots (%.1f MB staging): %.2f ms (%.2f Gpx/s)\n", chunks, slots,
                        blk * 2.0 * slots / 1e6, best * 1e3, N / best / 1e9);
            for (auto& e : ev) cudaEventDestroy(e);
            cudaFreeHost(ring);
            cudaFree(dblk);
        }
    }
    std::printf("check %d %d\n", h32[0][12345], h32[3][N - 1]);
    return 0;
}
