/*
 * sobel5_oracle.h -- CPU restatement of the reference's 4-direction 5x5
 * Sobel path, used ONLY as a test checker.
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library, and only as the
 * checker or the CPU timing arm.  The product path (libsobel5_b200.so) never
 * links, loads or calls it.
 *
 * Parity pinning: validated against (1) the SPEC.md per-op examples, (2) the
 * FNV-1a golden hashes of SURVEY.md Appendix A.3, and (3) outputs of the
 * reference headers themselves compiled by oracle/Makefile into
 * oracle/_ref/libsobel5_ref.so (tests/test_oracle.py).
 *
 * All functions are plain C over row-major, tightly packed planes (stride ==
 * width), exactly like sobel5::Plane (plane.hpp:14-63).
 */
#ifndef SOBEL5_ORACLE_H
#define SOBEL5_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* POD copy of sobel5::StreamTaps (pipeline.hpp:57-73). Same field order as
 * sobel5_taps in include/sobel5_gpu.h. */
typedef struct {
    int32_t a;
    int32_t f[5], h[5], k0[5], k1[5], gx_v[5], gy_v[5], gdm_f[5], gdm_d[5];
    int32_t wide_vagg;
} oracle_taps;

/* Mirror of sobel5::OpCounters (pipeline.hpp:26-51). */
typedef struct {
    uint64_t row_conv5_f, row_conv5_h, row_conv5_k0, row_conv5_k1;
    uint64_t row_diff, row_conv3_f, row_conv3_h, mac;
} oracle_counters;

/* Integer-parameter restatement of materialize() (filter_algebra.hpp:82-134,
 * 192-199). dir: 0=X 1=Y 2=D 3=DT.  k is 25 int32 row-major. */
void oracle_materialize(int64_t a, int64_t b, int64_t m, int64_t n, int dir, int32_t k[25]);

/* make_stream_taps() for integer (a,b,m,n) (pipeline.hpp:75-107). */
void oracle_make_stream_taps(int64_t a, int64_t b, int64_t m, int64_t n, oracle_taps* t);

/* conv2d_valid(GrayPlane, Kernel5) (oracle.hpp:19-33): valid-mode
 * correlation, int64 accumulator cast to int32.  out is (w-4)*(h-4). */
int oracle_conv2d_valid(const uint8_t* img, int w, int h, const int32_t k[25], int32_t* out);
/* conv2d_valid(GrayPlane, Kernel3): oracle.hpp:35-49. */
int oracle_conv2d_valid3(const uint8_t* img, int w, int h, const int32_t k[9], int32_t* out);

/* sobel5_4d() (oracle.hpp:82-98).  Any output pointer may be NULL. */
int oracle_sobel5_4d(const uint8_t* img, int w, int h, int64_t a, int64_t b, int64_t m,
                     int64_t n, int32_t* gx, int32_t* gy, int32_t* gd, int32_t* gdt,
                     double* g);

/* The arithmetic contract of run_stream(img, StreamTaps, ...) for ARBITRARY
 * (possibly fault-injected) taps (pipeline.hpp:304-414, 117-189, 268-282),
 * restated per output pixel rather than as a streaming schedule:
 *   F/H/K0/K1 = row_conv5 with f/h/k0/k1, D = p3 - p1           (:117-127)
 *   gx = sum gx_v[i] F(y+i),  gy = sum gy_v[i] H(y+i)           (:136-150)
 *   M  = sum gdm_f[i] F(y+i) - sum gdm_d[i] D(y+i)              (:166-189)
 *   P  = K0(y) + K1(y+1) - K1(y+3) - K0(y+4)                    (:152-164)
 *   gd = (P+M)/2, gdt = (P-M)/2, odd P+M -> ParityViolation      (:268-282)
 *   g  = sqrt(((gx^2+gy^2)+gd^2)+gdt^2) in double               (:401-407)
 * All 32-bit sums wrap mod 2^32, which equals both the int32 path and the
 * int64 (wide_vagg) path followed by the int32 narrowing cast.
 * Returns 0, 1 = ImageTooSmall, 3 = ParityViolation (first offending pair in
 * bad_sum / bad_diff when non-NULL). Any output may be NULL. */
int oracle_run_stream(const uint8_t* img, int w, int h, const oracle_taps* t, int32_t* gx,
                      int32_t* gy, int32_t* gd, int32_t* gdt, double* g, int32_t* bad_sum,
                      int32_t* bad_diff);

/* detail::quantize(plane, clamp_abs) for a RealPlane (image_io.hpp:235-240). */
void oracle_clamp_abs_f64(const double* g, size_t count, uint8_t* out);

/* synth_random (synth.hpp:11-35). */
void oracle_synth_random(uint8_t* img, int w, int h, uint64_t seed);

/* OpCounters that run_stream fills for a plan of the given strip widths
 * (pipeline.hpp:304-414 tallies, :416-445 summation), computed by walking
 * the reference schedule. prefetch: 0 = off, 1 = on. */
void oracle_stream_counters(int h, const int* strip_out_w, int n_strips, const oracle_taps* t,
                            int prefetch, oracle_counters* c);

/* ---- detect path ---- */

/* pad_replicate (image_io.hpp:279-291); out is (w+2r) x (h+2r).
 * Returns 0, 20 = EmptyPlane, 19 = DimMismatch (r < 0). */
int oracle_pad_replicate(const uint8_t* img, int w, int h, int r, uint8_t* out);

/* detail::quantize(plane, SaveMode::normalize) (image_io.hpp:242-255). */
void oracle_normalize_f64(const double* v, size_t n, uint8_t* out);
void oracle_normalize_i32(const int32_t* v, size_t n, uint8_t* out);
/* detail::quantize(SignedPlane, SaveMode::clamp_abs) (image_io.hpp:235-240). */
void oracle_clamp_abs_i32(const int32_t* v, size_t n, uint8_t* out);

/* sobel3_2d (oracle.hpp:58-70); out (w-2) x (h-2). Returns 0 or 1 (too small). */
int oracle_sobel3_2d(const uint8_t* img, int w, int h, int32_t* gx, int32_t* gy, double* g);

/* OpCounters of run_stream_3x3 (pipeline.hpp:488-547). */
void oracle_stream3_counters(int h, const int* strip_out_w, int n_strips, int prefetch,
                             oracle_counters* c);

/* FNV-1a 64 over raw bytes (SURVEY.md Appendix A.3 hashing convention). */
uint64_t oracle_fnv1a64(const void* data, size_t bytes);

#ifdef __cplusplus
}
#endif
#endif
