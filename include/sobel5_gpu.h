/*
 * sobel5_gpu.h -- C ABI of the B200-native 4-direction 5x5 Sobel path.
 *
 * This is the drop-in boundary for the reference's streaming engine
 * sobel5::run_stream (reference proj/include/sobel5/pipeline.hpp:452-477).
 * Every entry point takes plain pointers and sizes; no C++ or torch types
 * cross it, and nothing here throws.  The C++ API mirror
 * (include/sobel5_b200/sobel5.hpp) rethrows the reference's exception types
 * from the status codes; Python binds it with ctypes
 * (paper_2305_00515_b200/_abi.py).  See INTEGRATION.md for the bindings a
 * maintainer of the reference would add.
 *
 * Output contract (reference StreamResult, pipeline.hpp:284-291): four
 * int32 gradient planes gx, gy, gd, gdt and the double magnitude g, each
 * (W-4) x (H-4), valid-mode correlation.  Two optional extra planes are
 * available: g32 (float magnitude, correctly rounded sqrt of the exact sum)
 * and u8 (the clamp_abs edge map of image_io.hpp:235-240).  Any plane
 * pointer may be NULL; only the non-NULL planes are written.
 */
#ifndef SOBEL5_GPU_H
#define SOBEL5_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SOBEL5_GPU_ABI_VERSION 1

/* Status codes.  Each maps to one reference exception type
 * (reference errors.hpp:9-32); the C++ mirror throws that type. */
typedef enum sobel5_status {
    SOBEL5_OK = 0,
    SOBEL5_IMAGE_TOO_SMALL = 1,     /* ImageTooSmall     pipeline.hpp:454-456   */
    SOBEL5_DIM_MISMATCH = 2,        /* DimMismatch       pipeline.hpp:457-460   */
    SOBEL5_PARITY_VIOLATION = 3,    /* ParityViolation   pipeline.hpp:268-273   */
    SOBEL5_INVALID_ARG = 4,         /* null / misaligned pointer, bad pitch     */
    SOBEL5_CUDA_ERROR = 5,          /* CUDA runtime error (message via ctx)     */
    SOBEL5_OUT_OF_MEMORY = 6,       /* device or pinned allocation failed       */
    SOBEL5_NON_POSITIVE_PARAM = 7,  /* NonPositiveParam  filter_algebra.hpp:158 */
    SOBEL5_PARAM_OVERFLOW = 8,      /* ParamOverflow     filter_algebra.hpp:185 */
    SOBEL5_LANE_TOO_NARROW = 9,     /* LaneTooNarrow     strips.hpp:40-42       */
    SOBEL5_NO_DEVICE = 10,          /* no CUDA device: the path never falls back */
    SOBEL5_EMPTY_PLANE = 11         /* EmptyPlane        image_io.hpp:280         */
} sobel5_status;

/* POD copy of sobel5::StreamTaps (pipeline.hpp:57-73).  The kernels honour
 * arbitrary caller-supplied taps (e.g. the CLI's fault injection,
 * sobel5_cli.cpp:219); wide_vagg is accepted and ignored because 32-bit
 * wrapping arithmetic gives the int64 path's result after its int32 cast. */
typedef struct sobel5_taps {
    int32_t a;
    int32_t f[5];     /* -1, -b, 0, b, 1                */
    int32_t h[5];     /*  1,  n, m, n, 1                */
    int32_t k0[5];    /* a * (-m, -(n+b), -2, -(n+b), -m) */
    int32_t k1[5];    /* a * (b-n, -mb, -2nb, -mb, b-n) */
    int32_t gx_v[5];  /* a * (1, n, m, n, 1) on F rows  */
    int32_t gy_v[5];  /* a * (-1, -b, 0, b, 1) on H rows */
    int32_t gdm_f[5]; /* a * (m, n+b, 2, n+b, m) on F rows */
    int32_t gdm_d[5]; /* subtracted coefficients on D rows */
    int32_t wide_vagg;
} sobel5_taps;

/* Output planes.  All planes share one row stride `pitch`, in ELEMENTS.
 * Device entry points require: pitch >= width-4, pitch % 4 == 0, and every
 * non-NULL plane 32-byte aligned.  sobel5_run_host takes tightly packed host
 * planes (pitch == width-4, any alignment). */
typedef struct sobel5_planes {
    int32_t* gx;
    int32_t* gy;
    int32_t* gd;
    int32_t* gdt;
    double* g;
    float* g32;
    uint8_t* u8;
    int64_t pitch;
} sobel5_planes;

/* Diagnostics set by the kernels (nullable; device copies 16-byte aligned).
 * Zero it before the launch (strip_w may be set); violations != 0 means some
 * pixel had an odd P+M (recover_diag, pipeline.hpp:268-273) and (sum, diff)
 * is the pair the reference's run_stream with workers = 1 reports: the
 * first odd pixel in strip order (strips of strip_w output columns, i.e. the
 * plan's lane_width - 4; 0 = one strip), then row, then column
 * (run_strips_parallel, pipeline.hpp:416-445), frames first to last.
 * order is that pixel's position key (internal; 0 = none); order, sum and
 * diff are updated together as one 16-byte word.  The host entry points take
 * strip_w from *diag_out on entry. */
typedef struct sobel5_diag {
    int32_t violations;
    int32_t strip_w;
    int32_t reserved[2];
    uint64_t order;
    int32_t sum;
    int32_t diff;
} sobel5_diag;

/* Reference-schedule tallies (sobel5::OpCounters, pipeline.hpp:26-51). */
typedef struct sobel5_counters {
    uint64_t row_conv5_f, row_conv5_h, row_conv5_k0, row_conv5_k1;
    uint64_t row_diff, row_conv3_f, row_conv3_h, mac;
} sobel5_counters;

/* Per-frame scratch of the normalize export (image_io.hpp:242-255).
 * minmax: order-preserving keys of the smallest / largest value
 * (key(v) = bits(v) ^ (v < 0 ? ~0 : 1 << 63) for a double v, compared as
 * unsigned 64-bit integers); filled by pass 1, initialised by the library.  norm_table: the exact
 * piecewise-constant map S -> u8 of pass 2 for integer sums of squares
 * (thr[k] = smallest S whose normalized value is >= k), plus a float
 * estimate (lo_f, scale_f) used to seed the lookup. */
typedef struct sobel5_minmax {
    uint64_t lo_key;
    uint64_t hi_key;
} sobel5_minmax;

typedef struct sobel5_norm_table {
    double lo;          /* min g */
    double span;        /* max g - min g */
    float lo_f;         /* (float) lo */
    float scale_f;      /* (float) (255 / span), 0 if span <= 0 */
    uint32_t exact_s;   /* 1: thresholds valid (integer S), 0: use lo/span directly */
    uint32_t one_step;  /* 1: the float index estimate is within 1/4 step (one-compare map) */
    uint32_t thr[257];  /* thr[0] = 0, thr[256] = UINT32_MAX */
    uint32_t pad2_[3];
} sobel5_norm_table;

typedef struct sobel5_ctx sobel5_ctx; /* opaque: device, streams, buffers */

/* ---- library ------------------------------------------------------------- */
int sobel5_abi_version(void);
const char* sobel5_status_string(int status);
/* Number of kernel launches this process has issued through the library. */
uint64_t sobel5_launch_count(void);

/* Geometry the calling thread's last 5x5 stencil launch chose (diagnostics:
 * lets tests assert which code path a configuration takes).  band = output
 * rows per CTA, tma_load = 1 when the CTA's band rows came in by TMA bulk
 * copies, kernel = sobel5_kernel_for_taps of the taps, grid = CTA grid. */
typedef struct sobel5_launch_info {
    int band;
    int tma_load;
    int kernel;
    int grid_x, grid_y, grid_z;
} sobel5_launch_info;
sobel5_status sobel5_last_launch(sobel5_launch_info* out);

/* ---- host-only helpers (no GPU needed) ------------------------------------ */

/* make_stream_taps (pipeline.hpp:75-107) for integer (a, b, m, n), with the
 * validate_params rules that apply to integers (filter_algebra.hpp:157-188):
 * a >= 1 and b, m, n > 0 (NON_POSITIVE_PARAM), max |weight| <= 2^15
 * (PARAM_OVERFLOW). Rational parameters are validated by the C++ mirror. */
sobel5_status sobel5_make_taps(int64_t a, int64_t b, int64_t m, int64_t n, sobel5_taps* out);

/* OpCounters the reference's run_stream reports for a plan whose strips have
 * the given output widths (closed form of run_strip's tallies,
 * pipeline.hpp:304-414). prefetch: 0 off, 1 on. */
sobel5_status sobel5_plan_counters(int height, const int* strip_out_w, int n_strips,
                                   const sobel5_taps* taps, int prefetch, sobel5_counters* out);

/* ---- device entry points (caller-owned device memory, asynchronous) ------- */

/* One image.  d_in: width x height uint8, row stride in_pitch bytes
 * (in_pitch >= width rounded up to 4, in_pitch % 16 == 0, d_in 16-byte
 * aligned).  prefetch selects the kernel variant (reference Prefetch,
 * pipeline.hpp:21): 0 = direct loads, 1 = software-pipelined row prefetch.
 * stream is a cudaStream_t (NULL = legacy default stream).  Returns after
 * the launch is enqueued. */
sobel5_status sobel5_launch(const uint8_t* d_in, int64_t in_pitch, int width, int height,
                            const sobel5_taps* taps, int prefetch, const sobel5_planes* d_out,
                            sobel5_diag* d_diag, void* stream);

/* n_frames images of the same size in one launch: frame i starts at
 * d_in + i*in_frame_stride bytes and its planes at element offset
 * i*out_frame_stride (batched 1080p, config C4). */
sobel5_status sobel5_launch_batch(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                                  int width, int height, int n_frames, const sobel5_taps* taps,
                                  int prefetch, const sobel5_planes* d_out,
                                  int64_t out_frame_stride, sobel5_diag* d_diag, void* stream);

/* Row band of a row-partitioned image (config C5).  The band owns input
 * rows [0, band_rows) of d_in; the two rows above it come from d_top (NULL at
 * the image top) and the two below from d_bot (NULL at the image bottom).
 * d_top / d_bot may point into a PEER GPU's buffer (CUDA IPC / P2P mapped),
 * in which case the halo crosses NVLink inside the kernel, with no separate
 * exchange.  The output rows written are the valid centre rows of the
 * stacked image [top; band; bot], i.e. (rows_total - 4) rows starting at the
 * first centre row. */
sobel5_status sobel5_launch_band(const uint8_t* d_top, const uint8_t* d_in, const uint8_t* d_bot,
                                 int64_t in_pitch, int width, int band_rows,
                                 const sobel5_taps* taps, int prefetch,
                                 const sobel5_planes* d_out, sobel5_diag* d_diag, void* stream);

/* ---- detect path (sobel5_cli.cpp:127-189) ---------
 * pad = 1 fuses pad_replicate(img, 2) (image_io.hpp:279-291) into the
 * stencil's loads: the planes are then width x height (same size as the
 * input) and equal run_stream(pad_replicate(img, 2).plane, ...); an empty
 * image gives SOBEL5_EMPTY_PLANE.  pad = 0 is sobel5_launch_batch. */
sobel5_status sobel5_launch_ex(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                               int width, int height, int n_frames, const sobel5_taps* taps,
                               int prefetch, int pad, const sobel5_planes* d_out,
                               int64_t out_frame_stride, sobel5_diag* d_diag, void* stream);

/* Bytes of device scratch the normalize export needs (256-byte aligned):
 * per-frame min/max and threshold table plus a uint32 plane of the exact
 * integer g^2 with the output planes' pitch / frame stride (elements).
 * sobel5_quantize_plane needs sobel5_detect_scratch_bytes(0, 0, 0, 1). */
size_t sobel5_detect_scratch_bytes(int out_h, int64_t pitch, int64_t out_frame_stride,
                                   int n_frames);

/* The detect export: u8 = quantize(g, save_mode) (image_io.hpp:233-256) of
 * the (optionally padded) image; save_mode 0 = clamp_abs, 1 = normalize
 * (the CLI default, sobel5_cli.cpp:177).  d_out->u8 is required; any other
 * non-NULL plane of d_out is written too (the --dump-planes source).
 * normalize runs pass 1 (stencil: planes, per-frame min/max of g and, for
 * integer magnitudes, the g^2 plane into scratch), a threshold table, and
 * pass 2 (u8 from the g^2 plane through the table; non-integer magnitudes
 * re-run the stencil instead); bit-exact with the reference's double
 * arithmetic. */
sobel5_status sobel5_detect(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                            int width, int height, int n_frames, const sobel5_taps* taps,
                            int prefetch, int pad, int save_mode, const sobel5_planes* d_out,
                            int64_t out_frame_stride, void* d_scratch, sobel5_diag* d_diag,
                            void* stream);

/* detail::quantize of a device plane (save_plane, image_io.hpp:258-268):
 * kind 0 = RealPlane (double), 1 = SignedPlane (int32), 2 = GrayPlane
 * (uint8); pitch in elements,
 * u8_pitch in bytes; save_mode as above. */
sobel5_status sobel5_quantize_plane(const void* d_plane, int kind, int64_t pitch, int width,
                                    int height, int save_mode, uint8_t* d_u8, int64_t u8_pitch,
                                    void* d_scratch, void* stream);

/* synth_random (synth.hpp:20-35) generated on the device, optionally masked
 * (SURVEY.md section 8d inputs).  Pixel i of row-major order is byte i%8 of
 * splitmix64 word i/8; row_offset lets a band generate its slice. */
sobel5_status sobel5_synth_random_device(uint8_t* d_img, int64_t pitch, int width, int height,
                                         int64_t row_offset, uint64_t seed, uint8_t mask,
                                         void* stream);

/* ---- peer (CUDA IPC) mapping for row bands across GPUs -------------------
 * One rank exports the device buffer of its band; a neighbour imports it and
 * passes the imported pointer (plus row offsets) as d_top / d_bot of
 * sobel5_launch_band, so the 2-row halos are read over NVLink inside the
 * kernel.  d_ptr may point anywhere inside an allocation. */
typedef struct sobel5_ipc_handle {
    unsigned char bytes[64]; /* cudaIpcMemHandle_t of the containing allocation */
    int64_t offset;          /* byte offset of the exported pointer inside it */
} sobel5_ipc_handle;

sobel5_status sobel5_ipc_export(const void* d_ptr, sobel5_ipc_handle* out);
/* Maps a peer's exported buffer into this process (current device). */
sobel5_status sobel5_ipc_import(const sobel5_ipc_handle* h, const void** d_ptr);
sobel5_status sobel5_ipc_release(const void* d_ptr);

/* Mirrors the reference's own path choice for wide taps (make_stream_taps'
 * wide_vagg flag, pipeline.hpp:94-105, selecting the int64 vagg path).
 * Which kernel family serves these taps: 0 packed int16 lanes with the
 * default (1, 2, 6, 4) algebra compiled in, 1 packed int16 lanes with
 * runtime taps (every response < 2^15), 2 packed FP32 with runtime taps
 * (every partial sum < 2^22), 3 generic 32-bit wrapping kernel (any taps);
 * -1 for NULL.  Host-only, no device needed. */
int sobel5_kernel_for_taps(const sobel5_taps* taps);

/* ---- diagnostics ----------------------------------------------------------
 * Device self-check of the epilogue arithmetic over every integer S in
 * [lo, hi): which = 0 compares the kernels' double sqrt with IEEE
 * __dsqrt_rn((double)S); which = 1 compares the uint8 clamp_abs shortcut with
 * min(255, round(sqrt(S))); which = 2 checks the packed-float u8 epilogue
 * of the u8-only kernels on every integer S <= 65280 in range, and which = 3
 * on every float S >= 65281 whose bit pattern is in [lo, hi) (expects 255);
 * which = 4 / 5 do the same for the sqrt + saturating round of the u8-only
 * kernel (sobel5_u8.cuh).  Adds the number of mismatches to *d_count (device pointer, unsigned
 * 64-bit). */
sobel5_status sobel5_selftest(int which, uint32_t lo, uint32_t hi, uint64_t* d_count,
                              void* stream);

/* ---- context: host-buffer path (what the C++ run_stream wrapper calls) ---- */

sobel5_status sobel5_ctx_create(sobel5_ctx** out, int device);
void sobel5_ctx_destroy(sobel5_ctx* ctx);
/* (No reference counterpart: the reference allocates per call,
 * pipeline.hpp:462-467.)  Releases the context's cached device buffers and
 * pinned host staging
 * (kept across calls so repeated calls allocate nothing); no-op while a
 * begin/finish pair is pending. */
void sobel5_ctx_trim(sobel5_ctx* ctx);
/* Message of the last CUDA error seen by this context ("" if none). */
const char* sobel5_ctx_last_error(const sobel5_ctx* ctx);
/* Output columns per strip of the caller's StripPlan (lane_width - 4; 0 =
 * one strip, the default): orders the ParityViolation pair the host calls
 * report like the reference's run_stream with workers = 1 (sobel5_diag). */
sobel5_status sobel5_ctx_set_strip_width(sobel5_ctx* ctx, int strip_w);
/* Bytes of result planes the last sobel5_run_host / _begin / sobel3 host
 * call moved device -> host (the int16 wire included), for accounting. */
uint64_t sobel5_ctx_last_d2h_bytes(const sobel5_ctx* ctx);

/* Replaces sobel5::run_stream (pipeline.hpp:452-477: validation :454-460,
 * plane allocation :462-467, strip dispatch :416-445) for host buffers.
 * Synchronous end-to-end call: host image in (tightly packed W x H), host
 * planes out (tightly packed, pitch == width-4; NULL planes skipped).
 * Copies are chunked by row bands over pinned staging and overlapped with
 * the kernels on the context's streams.  On SOBEL5_PARITY_VIOLATION the
 * offending pair is returned in *diag_out (nullable). */
sobel5_status sobel5_run_host(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                              const sobel5_taps* taps, int prefetch, const sobel5_planes* h_out,
                              sobel5_diag* diag_out);

/* Split form of sobel5_run_host (same reference interface, pipeline.hpp:452)
 * for callers that allocate their result
 * planes while the device works (the C++ run_stream does): _begin enqueues
 * upload, kernels and downloads into the context's pinned staging and
 * returns; _finish waits chunk by chunk and copies the planes selected by
 * plane_mask (bit i = gx, gy, gd, gdt, g, g32, u8) into h_out, whose
 * non-NULL planes must match the mask exactly (pitch == width-4), or with
 * h_out = NULL only completes the call.  One
 * begin/finish pair at a time per context; sobel5_run_host in between
 * returns SOBEL5_INVALID_ARG.  Pageable destinations anywhere in this API go
 * through pinned staging plus a small host thread pool; page-locked ones
 * (cudaMallocHost / cudaHostRegister) are DMA'd directly.  Staging is capped
 * per context (env SOBEL5_STAGING_MAX_MB, default 4096): beyond it
 * sobel5_run_host downloads straight into pageable memory and _begin
 * returns SOBEL5_OUT_OF_MEMORY (use sobel5_run_host). */
/* A stream of n_frames W x H frames end to end (run_stream per frame,
 * pipelined across frames: frame f+1's upload and kernel overlap frame f's
 * download and host-side widening; 4 units in flight).  h_in: frame f at
 * h_in + f * in_frame_stride bytes (>= W*H, tightly packed rows); h_out:
 * planes with pitch W-4, frame f at + f * out_frame_stride elements
 * (>= (W-4)*(H-4)).  Same plane rules, wire and errors as sobel5_run_host;
 * diag_out covers every frame. */
sobel5_status sobel5_run_host_frames(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                                     int n_frames, int64_t in_frame_stride, const sobel5_taps* taps,
                                     int prefetch, const sobel5_planes* h_out,
                                     int64_t out_frame_stride, sobel5_diag* diag_out);
sobel5_status sobel5_run_host_begin(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                                    const sobel5_taps* taps, int prefetch, unsigned plane_mask);
sobel5_status sobel5_run_host_finish(sobel5_ctx* ctx, const sobel5_planes* h_out,
                                     sobel5_diag* diag_out);
/* Between _begin and _finish the staged planes can also be consumed as
 * they arrive: _chunk blocks until row chunk `chunk` (0, 1, ... while it
 * returns SOBEL5_OK) of every plane is in staging and gives its output rows
 * [*y0, *y1); _staging is the pinned, tightly packed plane i of the mask
 * (NULL otherwise).  Both may be called from several host threads.  Then
 * _finish with h_out = NULL completes the call (status, diag) without
 * copying. */
sobel5_status sobel5_run_host_chunk(sobel5_ctx* ctx, int chunk, int* y0, int* y1);
/* The same split form for the 3x3 operator (run_stream_3x3): planes gx, gy,
 * g, g32, u8 (mask bits 0, 1, 4, 5, 6; gd / gdt bits are rejected), then
 * _chunk / _staging / _finish as above with pitch == width-2. */
sobel5_status sobel3_run_host_begin(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                                    int prefetch, unsigned plane_mask);
const void* sobel5_run_host_staging(const sobel5_ctx* ctx, int plane);
/* Bytes per element of staged plane i of the pending call (0 if not in the
 * mask).  With default taps and exactly the StreamResult planes (mask 0x1f)
 * gx, gy, gd, gdt cross PCIe as int16 (every value lies in [-2^15, 2^15);
 * env SOBEL5_WIRE16=0 disables it): sobel5_run_host widens them into the
 * caller's int32 planes itself; in the split _begin form their staging holds
 * int16 (2) and the consumer sign-extends (_finish with h_out widens). */
int sobel5_run_host_staging_elem(const sobel5_ctx* ctx, int plane);

/* ---- the classic 3x3 two-direction operator ---------
 * run_stream_3x3 (pipeline.hpp:551-573) / sobel3_2d (oracle.hpp:58-70):
 * gx, gy int32 and g double (plus optional g32 / u8 clamp_abs) of a valid
 * (W-2) x (H-2) output, or W x H with pad = 1 (pad_replicate(img, 1)).
 * d_out->gd and ->gdt must be NULL.  Images below 3x3 give
 * SOBEL5_IMAGE_TOO_SMALL (pipeline.hpp:553-556). */
sobel5_status sobel3_launch(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                            int width, int height, int n_frames, int prefetch, int pad,
                            const sobel5_planes* d_out, int64_t out_frame_stride, void* stream);

/* Detect with --op sobel3_2d (sobel5_cli.cpp:128-149): u8 = quantize(g). */
sobel5_status sobel3_detect(const uint8_t* d_in, int64_t in_pitch, int64_t in_frame_stride,
                            int width, int height, int n_frames, int prefetch, int pad,
                            int save_mode, const sobel5_planes* d_out, int64_t out_frame_stride,
                            void* d_scratch, void* stream);

/* OpCounters of run_stream_3x3 (pipeline.hpp:488-547) for a plan. */
sobel5_status sobel3_plan_counters(int height, const int* strip_out_w, int n_strips, int prefetch,
                                   sobel5_counters* out);

/* Host-buffer run_stream_3x3: tightly packed planes (pitch == width-2). */
sobel5_status sobel3_run_host(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                              int prefetch, const sobel5_planes* h_out);

/* Host-buffer detect (what the CLI's detect command needs): tightly packed
 * W x H input, h_u8 receives the (out_w x out_h) edge map, h_planes
 * (nullable, pitch == out_w) any planes to dump.  out = W x H with pad = 1,
 * (W-4) x (H-4) otherwise. */
sobel5_status sobel5_detect_host(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                                 const sobel5_taps* taps, int prefetch, int pad, int save_mode,
                                 uint8_t* h_u8, const sobel5_planes* h_planes,
                                 sobel5_diag* diag_out);

/* Host-buffer detail::quantize (save_plane's export, image_io.hpp:233-268):
 * tightly packed plane (kind 0 double, 1 int32, 2 uint8), h_u8 same size. */
sobel5_status sobel5_quantize_host(sobel5_ctx* ctx, const void* h_plane, int kind, int width,
                                   int height, int save_mode, uint8_t* h_u8);

/* ---- the oracle's dense correlation (oracle.hpp:19-49) ------------------
 * conv2d_valid(img, Kernel5 / Kernel3): valid-mode correlation (no kernel
 * flip) of a uint8 image with an arbitrary ksize x ksize int32 kernel
 * (`kernel` is a HOST array, row-major), int32 result equal to the
 * reference's int64 sum cast to int32.  ksize is 5 or 3; images smaller
 * than the kernel give SOBEL5_IMAGE_TOO_SMALL.  d_in: in_pitch % 16 == 0,
 * 16-byte aligned; d_out: (W-k+1) x (H-k+1) with row stride out_pitch
 * elements. */
sobel5_status sobel5_conv2d_valid(const uint8_t* d_in, int64_t in_pitch, int width, int height,
                                  const int32_t* kernel, int ksize, int32_t* d_out,
                                  int64_t out_pitch, void* stream);
/* Host buffers (tightly packed W x H in, (W-k+1) x (H-k+1) out). */
sobel5_status sobel5_conv2d_valid_host(sobel5_ctx* ctx, const uint8_t* h_in, int width,
                                       int height, const int32_t* kernel, int ksize,
                                       int32_t* h_out);
/* sobel5_4d (oracle.hpp:82-98): the four dense 5x5 correlations with the
 * materialised kernels Kx, Ky, Kd, Kdt (`kernels`: HOST array of 4 x 25
 * int32, row-major, in that order) and the magnitude
 * sqrt(gx*gx + gy*gy + gd*gd + gdt*gdt) in double with the reference's
 * rounding sequence, all in one device pass -- the oracle's algorithm, not
 * the streaming one.  d_out->g32 and ->u8 must be NULL; other planes may be
 * NULL (skipped). */
sobel5_status sobel5_dense_4d(const uint8_t* d_in, int64_t in_pitch, int width, int height,
                              const int32_t* kernels, const sobel5_planes* d_out, void* stream);
/* Host buffers: tightly packed planes (pitch == width-4). */
sobel5_status sobel5_dense_4d_host(sobel5_ctx* ctx, const uint8_t* h_in, int width, int height,
                                   const int32_t* kernels, const sobel5_planes* h_out);

/* ---- one image row-band partitioned over several GPUs (config C5) --------
 * SURVEY.md 8b/8e; replaces the reference's strip thread pool
 * run_strips_parallel (pipeline.hpp:416-445) at device granularity.  One
 * process drives n bands; band k owns input rows [k*H/n, (k+1)*H/n) on
 * devices[k] and writes the output rows centred in it (no gather: output
 * rows are disjoint).  devices may repeat (several bands on one GPU).
 * Halo transport: PEER -- the band kernel reads the neighbours' 2 rows from
 * their HBM over NVLink inside the stencil (needs peer access); COPY -- the
 * 2-row halos are copied device to device while the interior computes, then
 * two 2-row seams; AUTO -- PEER where every neighbour pair has peer access.
 * Ordering uses events on the bands' streams only (no host barrier):
 * run_bands waits for everything already enqueued on each band's stream
 * before reading that band's rows, and afterwards every band's stream waits
 * until its neighbours' kernels are done, so input rows the caller writes
 * next on a band's stream never race the halo reads of the previous call. */
enum { SOBEL5_MGPU_AUTO = -1, SOBEL5_MGPU_PEER = 0, SOBEL5_MGPU_COPY = 1 };

typedef struct sobel5_mgpu sobel5_mgpu; /* opaque */

typedef struct sobel5_band_info {
    int device;
    int r0, r1;         /* input rows [r0, r1) of the image held by the band */
    int out_row0;       /* first row of the (W-4) x (H-4) output it writes */
    int out_rows;       /* output rows it writes */
    uint8_t* d_in;      /* its input rows on `device`, row stride in_pitch */
    int64_t in_pitch;
    void* stream;       /* cudaStream_t of the band (on `device`) */
    int transport;      /* SOBEL5_MGPU_PEER or _COPY (AUTO resolved) */
} sobel5_band_info;

/* Errors: IMAGE_TOO_SMALL below 5x5, DIM_MISMATCH when a band would get
 * fewer than 4 rows, INVALID_ARG for a bad device or PEER without peer
 * access, NO_DEVICE without a GPU. */
sobel5_status sobel5_mgpu_create(sobel5_mgpu** out, const int* devices, int n, int width,
                                 int height, int transport);
void sobel5_mgpu_destroy(sobel5_mgpu* m);
sobel5_status sobel5_mgpu_band(const sobel5_mgpu* m, int k, sobel5_band_info* info);
/* Enqueue each band's rows of a tightly packed W x H host image (pinned
 * memory makes this asynchronous), or synth_random(W, H, seed) & mask
 * generated on every band's device. */
sobel5_status sobel5_mgpu_upload(sobel5_mgpu* m, const uint8_t* h_img);
sobel5_status sobel5_mgpu_synth(sobel5_mgpu* m, uint64_t seed, uint8_t mask);
/* Asynchronous: band k's output rows into d_out[k] (planes on devices[k],
 * out_rows x pitch, same plane rules as sobel5_launch). */
sobel5_status sobel5_mgpu_run_bands(sobel5_mgpu* m, const sobel5_taps* taps, int prefetch,
                                    const sobel5_planes* d_out);
sobel5_status sobel5_mgpu_sync(sobel5_mgpu* m);
/* Host buffers end to end (the multi-GPU run_stream): upload, bands, and
 * each band's rows downloaded over its own GPU's link into the tightly
 * packed host planes (pitch == width-4). */
sobel5_status sobel5_mgpu_run_host(sobel5_mgpu* m, const uint8_t* h_in, const sobel5_taps* taps,
                                   int prefetch, const sobel5_planes* h_out);
/* After run_host returned SOBEL5_PARITY_VIOLATION: the offending pair -- the
 * first odd pixel of the whole image in strip, row, column order (strips of
 * strip_w output columns, see sobel5_mgpu_set_strip_width; 0 = one strip),
 * as the reference's run_stream with workers = 1 reports it. */
sobel5_status sobel5_mgpu_last_diag(const sobel5_mgpu* m, sobel5_diag* out);
/* The strip width (plan lane width - 4) ordering run_host's ParityViolation
 * pair, like sobel5_ctx_set_strip_width. */
sobel5_status sobel5_mgpu_set_strip_width(sobel5_mgpu* m, int strip_w);

/* ---- stream-ordered flags (cross-process band ordering, bands.py) --------
 * host_register maps host memory (e.g. a shared-memory segment several
 * processes map) for device access; stream_write_u32 stores `value` to the
 * flag when the stream reaches it; stream_wait_u32 blocks the stream (not
 * the host) until (int32_t)(*flag - value) >= 0 (cuStreamWaitValue32 GEQ). */
sobel5_status sobel5_host_register(void* p, size_t bytes, void** d_ptr);
sobel5_status sobel5_host_unregister(void* p);
sobel5_status sobel5_stream_write_u32(uint32_t* d_flag, uint32_t value, void* stream);
sobel5_status sobel5_stream_wait_u32(const uint32_t* d_flag, uint32_t value, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SOBEL5_GPU_H */
