// pipe_rates.cu -- issue-rate probe for the instruction classes the u8
// (issue-bound) kernels use: warp-instructions per SMSP per cycle for each
// op alone and for pairs interleaved (do two pipes co-issue?).  One wave of
// 4 CTAs x 256 threads per SM, 8 independent chains per thread; cycles from
// clock64 inside each CTA.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o pipe_rates pipe_rates.cu; check the SASS with cuobjdump -sass.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

template <int OP>
__device__ __forceinline__ void step(uint32_t (&r)[8], float2 (&f)[8], float (&s)[8], uint32_t k) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int n = (j + 1) & 7;
        const bool odd = j & 1;
        if (OP == 0) r[j] = r[j] + r[n] + k;                             // IADD3
        if (OP == 1) r[j] = r[j] * 6u + r[n];                            // IMAD imm
        if (OP == 2) r[j] = __byte_perm(r[j], r[n], 0x5432);             // PRMT
        if (OP == 3) r[j] = (r[j] & r[n]) ^ k;                           // LOP3
        if (OP == 4) f[j] = ffma2(f[j], f[n], f[j]);                     // FFMA2 3-reg
        if (OP == 5) f[j] = ffma2(f[j], make_float2(2.f, 2.f), f[n]);    // FFMA2 imm
        if (OP == 6) f[j] = fadd2(f[j], f[n]);                           // FADD2
        if (OP == 7) f[j] = fmul2(f[j], f[n]);                           // FMUL2
        if (OP == 8) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(s[j]));   // MUFU.RSQ
        if (OP == 9) asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(s[j]));    // MUFU.SQRT
        if (OP == 10) {                                                   // F2I u8 sat
            uint32_t t;
            asm volatile("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(t) : "f"(s[j]));
            r[j] += t;
        }
        if (OP == 11) { if (odd) r[j] = r[j] * 6u + r[n]; else r[j] = r[j] + r[n] + k; }  // IMAD+IADD3
        if (OP == 12) { if (odd) f[j] = ffma2(f[j], f[n], f[j]); else r[j] = r[j] + r[n] + k; }
        if (OP == 13) { if (odd) f[j] = ffma2(f[j], f[n], f[j]); else r[j] = __byte_perm(r[j], r[n], 0x5432); }
        if (OP == 14) { if (odd) f[j] = fadd2(f[j], f[n]); else r[j] = r[j] + r[n] + k; }
        if (OP == 15) { if (odd) f[j] = ffma2(f[j], f[n], f[j]); else r[j] = r[j] * 6u + r[n]; }
        if (OP == 16) s[j] = fmaf(s[j], s[n], s[j]);                      // FFMA 3-reg
        if (OP == 17) s[j] = fmaf(s[j], 3.f, s[n]);                       // FFMA imm
        if (OP == 18) s[j] = s[j] + s[n];                                 // FADD
        if (OP == 19) { if (odd) f[j] = ffma2(f[j], make_float2(2.f, 2.f), f[n]); else r[j] = r[j] + r[n] + k; }
        if (OP == 20) { if (odd) s[j] = fmaf(s[j], 3.f, s[n]); else r[j] = r[j] + r[n] + k; }  // FFMA imm + IADD3
        if (OP == 21) { if (odd) r[j] = r[j] * 6u + r[n]; else r[j] = __byte_perm(r[j], r[n], 0x5432); }
        if (OP == 22) { if (odd) f[j] = fadd2(f[j], f[n]); else r[j] = __byte_perm(r[j], r[n], 0x5432); }
        if (OP == 23) {  // vmin/vmax s16x2
            asm volatile("min.s16x2 %0, %0, %1;" : "+r"(r[j]) : "r"(r[n]));
        }
        if (OP == 24) {  // HFMA2
            __half2 a = *reinterpret_cast<__half2*>(&r[j]);
            __half2 b = *reinterpret_cast<__half2*>(&r[n]);
            a = __hfma2(a, b, a);
            r[j] = *reinterpret_cast<uint32_t*>(&a);
        }
    }
}

template <int OP>
__global__ void __launch_bounds__(256) probe(uint32_t* sink, long long* cyc, int iters) {
    uint32_t r[8];
    float2 f[8];
    float s[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        r[j] = threadIdx.x * 7 + j;
        f[j] = make_float2(1.0f + 1e-7f * j, 1.0f - 1e-7f * threadIdx.x);
        s[j] = 1.0f + 1e-6f * (threadIdx.x + j);
    }
    const uint32_t k = static_cast<uint32_t>(iters) * 3u + 1u;
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < iters; ++i) step<OP>(r, f, s, k);
    __syncthreads();
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc ^= r[j] ^ __float_as_uint(f[j].x) ^ __float_as_uint(f[j].y) ^ __float_as_uint(s[j]);
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

#include <cuda_fp16.h>

template <int OP>
void run(const char* name, int sms, uint32_t* sink, long long* d_cyc, long long* h_cyc) {
    const int blocks = sms * 4, iters = 4096;
    probe<OP><<<blocks, 256>>>(sink, d_cyc, 64);
    probe<OP><<<blocks, 256>>>(sink, d_cyc, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h_cyc, d_cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int b = 0; b < blocks; ++b) mx = h_cyc[b] > mx ? h_cyc[b] : mx;
    // per SMSP: 8 warps (4 CTAs x 8 warps / 4 SMSPs) x iters x 8 instructions
    const double per_smsp = 8.0 * iters * 8.0;
    printf("%-28s %6.3f warp-instr/SMSP/clk  (%lld cycles)\n", name, per_smsp / mx, mx);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* sink;
    long long *d_cyc, h_cyc[4096];
    cudaMalloc(&sink, 1024 * 4);
    cudaMalloc(&d_cyc, 4096 * 8);
    printf("SMs %d\n", sms);
    run<0>("IADD3", sms, sink, d_cyc, h_cyc);
    run<1>("IMAD imm", sms, sink, d_cyc, h_cyc);
    run<2>("PRMT", sms, sink, d_cyc, h_cyc);
    run<3>("LOP3", sms, sink, d_cyc, h_cyc);
    run<4>("FFMA2 3-reg", sms, sink, d_cyc, h_cyc);
    run<5>("FFMA2 imm", sms, sink, d_cyc, h_cyc);
    run<6>("FADD2", sms, sink, d_cyc, h_cyc);
    run<7>("FMUL2", sms, sink, d_cyc, h_cyc);
    run<8>("MUFU.RSQ", sms, sink, d_cyc, h_cyc);
    run<9>("MUFU.SQRT", sms, sink, d_cyc, h_cyc);
    run<10>("F2I.U8.sat (+IADD)", sms, sink, d_cyc, h_cyc);
    run<11>("IMAD + IADD3", sms, sink, d_cyc, h_cyc);
    run<12>("FFMA2 + IADD3", sms, sink, d_cyc, h_cyc);
    run<13>("FFMA2 + PRMT", sms, sink, d_cyc, h_cyc);
    run<14>("FADD2 + IADD3", sms, sink, d_cyc, h_cyc);
    run<15>("FFMA2 + IMAD", sms, sink, d_cyc, h_cyc);
    run<16>("FFMA 3-reg", sms, sink, d_cyc, h_cyc);
    run<17>("FFMA imm", sms, sink, d_cyc, h_cyc);
    run<18>("FADD", sms, sink, d_cyc, h_cyc);
    run<19>("FFMA2 imm + IADD3", sms, sink, d_cyc, h_cyc);
    run<20>("FFMA imm + IADD3", sms, sink, d_cyc, h_cyc);
    run<21>("IMAD + PRMT", sms, sink, d_cyc, h_cyc);
    run<22>("FADD2 + PRMT", sms, sink, d_cyc, h_cyc);
    run<23>("VIMNMX.S16x2", sms, sink, d_cyc, h_cyc);
    run<24>("HFMA2", sms, sink, d_cyc, h_cyc);
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
