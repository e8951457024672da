/*
 * adct.h — C ABI of the B200 (sm_100a) hot path of arXiv 1402.6034,
 * "An orthogonal 8-point DCT approximation" (round-off approximation C0 = [2C],
 * orthogonalised by the diagonal S).
 *
 * Citations: P:n = PAPER.md line n (Section / equation named beside it).
 *
 * Notation:
 *   X    8x8 uint8 block, rows i (vertical), columns j (horizontal)
 *   T    = C0 = [2 C], the displayed {0,+-1} matrix
 *   d    = diag(T T^T) = (8,6,4,6,8,6,4,6); S = D = diag(d)^(-1/2)
 *   C    = S . C0, the proposed orthogonal approximation C_orth
 *   Y    = T . X . T^T, the integer coefficient block (22-addition butterfly    (P:250-283,
 *          per 1-D transform, Table 1), |Y| <= 16320 so int16 is exact          P:482-487)
 *   Z    = C . X . C^T = D . Y . D, Z_ij = Y_ij / sqrt(d_i d_j) (orthonormal domain)
 *   M_r  keep the first r coefficients of the standard zig-zag scan (1<=r<=64)
 *   X^   = C^T . (M_r . Z) . C, the reconstruction ("inverse procedure")
 *   S is folded into the zonal / quantisation step: the kernels use the
 *   integer weights W_ij = 576 / (d_i d_j) in {9,12,16,18,24,36}, so that
 *   576 X^ = T^T (W . M_r . Y) T is an exact integer.
 *   PSNR = 10 log10(255^2 / MSE), MSE = SSE / (h w)
 *
 * Layout (all entry points): n images of h x w pixels (h, w positive multiples of 8),
 * row-major; `pitch` = bytes between rows; `img_stride` = bytes between images.
 * Coefficient planes are image-shaped: coefficient (i, j) of the block at block
 * row by, block column bx is stored at pixel (8 by + i, 8 bx + j) (reading R12).
 *
 * Ownership: every pointer is a DEVICE pointer owned by the caller unless stated;
 * the library allocates nothing and keeps no mutable global state. All calls are
 * asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream); results
 * are valid once the stream is synchronised. Functions are re-entrant.
 *
 * Errors: arguments are validated before anything is enqueued. On ADCT_EINVAL /
 * ADCT_EALIGN nothing is enqueued. ADCT_ECUDA means a CUDA launch/driver error;
 * adct_last_cuda_error() returns its cudaError_t (thread-local).
 */
#ifndef ADCT_H
#define ADCT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* adct_stream_t; /* = cudaStream_t */

typedef enum {
  ADCT_OK = 0,
  ADCT_EINVAL = 1, /* n < 1, h or w not a positive multiple of 8, r outside [1,64], q < 0 or NaN,
                      pitch < row bytes, img_stride < h * pitch, unknown enum, NULL required pointer,
                      or more than 2^30 tiles of 16 x 256 pixels (4 TiB of uint8) in one call */
  ADCT_EALIGN = 2, /* a pointer not 16-byte aligned, or a pitch / image stride not a multiple of 16
                      (TMA global-address and stride rules) */
  ADCT_ECUDA = 3   /* CUDA launch or driver error; see adct_last_cuda_error() */
} adct_status;

typedef enum {
  ADCT_COEF_I16 = 0, /* int16 Y = T X T^T, exact (range [-8160, 16320])            */
  ADCT_COEF_I32 = 1, /* int32 Y = T X T^T, exact                                     */
  ADCT_COEF_F32 = 2  /* float Z = D Y D = C X C^T, one rounding: Y * fp32(1/sqrt(d_i d_j)) */
} adct_coef_t;

typedef enum {
  ADCT_RECON_NONE = 0, /* no reconstruction written                                    */
  ADCT_RECON_F32 = 1,  /* float X^ (unrounded, unclamped)                               */
  ADCT_RECON_U8 = 2    /* uint8 clamp(round_half_away(X^), 0, 255), decided on the exact 576 X^ */
} adct_recon_t;

/*
 * adct_forward — per 8x8 block, the 2-D forward transform T . X . T^T with the fast
 * algorithm of Fig. 1 / Table 1 on rows then columns; zig-zag
 * positions >= r are written as 0 (r = 64 keeps all).
 *   src   [n][h][pitch] uint8, 16-B aligned; pitch, img_stride multiples of 16.
 *   coef  image-shaped plane of coef_t; coef_pitch / coef_img_stride in bytes,
 *         multiples of 16, coef_pitch >= w * sizeof(element).
 * Returns ADCT_OK / EINVAL / EALIGN / ECUDA.
 */
adct_status adct_forward(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                         int64_t img_stride, int r, void* coef, adct_coef_t coef_t,
                         int64_t coef_pitch, int64_t coef_img_stride, adct_stream_t stream);

/*
 * adct_inverse — the inverse procedure: X^ = C^T (M_r . Z) C per block.
 * From ADCT_COEF_I16 / I32 (Y) the diagonal is folded as W / 576 (exact integers until the
 * final division while every node stays below 2^24; int32 values convert exactly to fp32 first);
 * from ADCT_COEF_F32 (Z) the kernel computes T^T (M_r . Z . s) T in fp32, and values at masked
 * positions (zig-zag >= r) are ignored even when they are NaN / Inf.  u8 output saturates:
 * clamp(round_half_away(X^), 0, 255) for any coefficient plane (decided on the integer 576 X^ for
 * I16 / I32, on the fp32 X^ for F32).
 *   coef  image-shaped coefficient plane (layout as adct_forward's output).
 *   dst   image-shaped reconstruction, dst_t = ADCT_RECON_F32 or ADCT_RECON_U8.
 */
adct_status adct_inverse(const void* coef, adct_coef_t coef_t, int64_t n, int64_t h, int64_t w,
                         int64_t coef_pitch, int64_t coef_img_stride, int r, void* dst,
                         adct_recon_t dst_t, int64_t dst_pitch, int64_t dst_img_stride,
                         adct_stream_t stream);

/*
 * adct_compress_psnr — the fused hot path: forward (22-add butterflies, rows then columns),
 * then either
 *   q == 0: ZONAL — keep the first r zig-zag coefficients, S folded as W;
 *   q  > 0: QUANT — D-scaled uniform quantiser on Z (reading R10): k = round_half_away(Z / q)
 *           for zig-zag positions < r (else 0), dequantise Z^ = q k,
 * then the inverse with C^T and the per-image squared error
 * sse[i] = sum over image i of (x - X^)^2 on the unrounded reconstruction (reading R3).
 *   src    [n][h][pitch] uint8 (as adct_forward).
 *   recon  optional (may be NULL with recon_t = ADCT_RECON_NONE) image-shaped reconstruction.
 *   sse    device double[n], OVERWRITTEN (the call zero-fills it on `stream` first).
 * Quantiser decision: k = round-to-nearest(Y * c) in one fp32 FMA, c the smallest fp32 strictly
 * above 1/(q sqrt(d_i d_j)); equal to the exact round-half-away decision for every reachable Y
 * when q = 16 (exhaustive check: tests/test_quant_decision.py).  With q > 0 and r < 64 the
 * coefficients at zig-zag positions >= r are discarded before quantisation (k = 0, reading R17).
 * Determinism: every per-image sum is accumulated on a fixed-point grid (2^-k pixel^2, k chosen per
 * call from h * w) from per-tile partials with integer atomics, so sse is bit-identical across
 * repeated calls, streams, graph replays and any split of the images across calls or ranks.
 * u8 reconstruction: clamp(round_half_away(X^), 0, 255) for every X^ (saturating; the zonal
 * decision is taken on the exact integer 576 X^, the quantiser's on the fp32 X^).
 * Launches: the kernel plus one small fixed-point -> fp64 conversion kernel.
 */
adct_status adct_compress_psnr(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                               int64_t img_stride, int r, float q, void* recon,
                               adct_recon_t recon_t, int64_t recon_pitch, int64_t recon_img_stride,
                               double* sse, adct_stream_t stream);

/*
 * adct_compress_sse576 — the zonal pass (q = 0) with the EXACT integer error sum:
 * sse576[i] = sum over image i of (576 x - R)^2, R = C0^T (W . M_r . Y) C0 (576 X^ = R),
 * every term an exact integer squared and summed in 64-bit integers (bit-exact; no fp rounding).
 * Same forward / mask / inverse as adct_compress_psnr with q = 0 (the runtime-mask kernel).
 *   sse576  device uint64_t[n], OVERWRITTEN.      sse  optional device double[n]: sse576 / 576^2.
 *   EINVAL additionally when h * w > 2^26 (the per-image sum must stay below 2^63, so the result is
 *   also exact as int64: |576 x - R| <= 329205).  A validation path: slower than
 *   adct_compress_psnr (64-bit multiply-adds per pixel).
 */
adct_status adct_compress_sse576(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                                 int64_t img_stride, int r, uint64_t* sse576, double* sse,
                                 adct_stream_t stream);

/*
 * adct_psnr — PSNR = 10 log10(255^2 * pixels / sse[i]), +inf when sse[i] == 0.
 *   sse, psnr  device double[count]; pixels = h * w of each image (> 0).
 */
adct_status adct_psnr(const double* sse, int64_t count, int64_t pixels, double* psnr,
                      adct_stream_t stream);

/*
 * adct_compress_psnr_multi — several zonal r over the same images (q = 0, SSE only):
 * sse[k * n + i] = adct_compress_psnr's SSE of image i at r = r_list[k] (OVERWRITTEN).
 * For BASELINE C5's set {1, 3, 6, 10, 15, 21, 28, 36} (any order) one fused kernel reads each tile
 * once, runs the forward once and, for every r, the zonal step, inverse and per-pixel error with
 * that r's own arithmetic (results identical to the single-r calls up to fp64 summation order);
 * any other set runs independent passes.  n_r in [1, 64]; sse device double[n_r * n].
 */
adct_status adct_compress_psnr_multi(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                                     int64_t img_stride, const int* r_list, int n_r, double* sse,
                                     adct_stream_t stream);

/*
 * adct_compress_psnr_host — end-to-end entry with HOST buffers: copies the images from host
 * memory (pinned recommended; host_src with host_pitch / host_img_stride in bytes) through the
 * caller's device staging buffer `dev_buf` (dev_buf_bytes >= one image of h * w bytes; images are
 * staged compactly, pitch = w rounded up to 16), compresses them for each of the n_r values
 * r_list[k] (q as adct_compress_psnr; with q = 0 the set {1, 3, 6, 10, 15, 21, 28, 36} runs as the
 * fused multi-r kernel of adct_compress_psnr_multi, other sets as independent passes), runs
 * adct_psnr, and copies PSNR back to host_psnr[k * n + i].
 *   dev_sse      device double[2 * n_r * n] scratch: SSE in [0, n_r n), PSNR in [n_r n, 2 n_r n).
 *   copy_stream  optional caller-owned stream (NULL: copies and passes alternate on `stream`).  With
 *                a copy stream, n >= 2 and dev_buf holding >= two images, the images are staged in
 *                chunks of about n / 8 through two halves of dev_buf on copy_stream, so the copy of
 *                chunk c+1 overlaps the passes of chunk c (ordered by events created and released by
 *                the call; no stream is created; the copy stream first waits for work already queued
 *                on `stream`).  Every variant is stream-ordered and can be captured into a CUDA graph.
 *   Asynchronous: host_psnr is valid after `stream` is synchronised.
 */
adct_status adct_compress_psnr_host(const uint8_t* host_src, int64_t n, int64_t h, int64_t w,
                                    int64_t host_pitch, int64_t host_img_stride,
                                    const int* r_list, int n_r, float q, uint8_t* dev_buf,
                                    int64_t dev_buf_bytes, double* dev_sse, double* host_psnr,
                                    adct_stream_t stream, adct_stream_t copy_stream);

/*
 * Dense comparator / variant path: the same block pipeline with an 8x8
 * transform T applied as dense fp32 matrix products (SSE in fp64) — for the paper's comparison curves
 * (Fig. 3): the exact DCT, the SDCT, the coarse C0/2, or any caller matrix.
 *   ADCT_T_PROPOSED  C_orth = S C0 (dense; cross-check of the fast path)
 *   ADCT_T_DCT       exact orthonormal DCT-II (reading R1)
 *   ADCT_T_SDCT      sign(C) / (2 sqrt 2) (reading R11; not orthogonal)
 *   ADCT_T_COARSE    C0 / 2 (not orthogonal)
 *   ADCT_T_CUSTOM    `custom`: host double[64], row-major
 * Per block Z = T X T^T, the first r zig-zag coefficients kept, X^ = T^T Z T (the transpose is the
 * exact inverse for orthogonal T and the approximate inversion otherwise), and
 * sse[i] = per-image sum of (x - X^)^2 in fp64 (sse: device double[n], overwritten).
 */
typedef enum {
  ADCT_T_PROPOSED = 0,
  ADCT_T_DCT = 1,
  ADCT_T_SDCT = 2,
  ADCT_T_COARSE = 3,
  ADCT_T_CUSTOM = 4,
  ADCT_T_CEIL = 5 /* F4 ("floor and ceiling functions can be considered instead of the
                     round-off function"): the orthogonal polar factor (T T^T)^(-1/2) T of
                     T = ceil(2 C) (entries {0, 1}, det 16; T T^T is not diagonal, so the
                     orthogonaliser is a dense symmetric matrix and there is no fast algorithm).
                     floor(2 C) is singular (its DC row floors to 0) and has no entry. */
} adct_transform_t;

adct_status adct_compress_psnr_dense(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                                     int64_t img_stride, int r, adct_transform_t t, const double* custom,
                                     float* recon /* nullable f32 plane */, int64_t recon_pitch,
                                     int64_t recon_img_stride, double* sse, adct_stream_t stream);

/*
 * adct_compress_psnr_sdct — the SDCT comparator (reading R11: sign(C) / (2 sqrt 2)) on the
 * INTEGER fast path: per block Y = T_s X T_s^T with T_s = sign(C) by the
 * 24-addition fast algorithm (Table 1) on packed 2 x int16 lanes (exact), the first r
 * zig-zag coefficients kept, the reconstruction X^ = R / 64 with R = T_s^T (M_r . Y) T_s by the
 * transposed 24-addition graph (exact integers in fp32), e = 64 x - R exact per pixel, and
 * sse[i] = per-image sum of (x - X^)^2 (deterministic fixed-point sum, as adct_compress_psnr).
 * The SDCT is not orthogonal: the transpose is its "approximate inversion".
 *   src as adct_forward;  sse device double[n], overwritten.
 */
adct_status adct_compress_psnr_sdct(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                                    int64_t img_stride, int r, double* sse, adct_stream_t stream);

/*
 * adct_uqi — universal quality index: per image, the mean over all
 * 8x8 sliding windows (stride 1) of Q = 4 s_xy mx my / ((s_x^2 + s_y^2)(mx^2 + my^2)) between
 * the uint8 original x and an f32 reconstruction y (e.g. ADCT_RECON_F32 of adct_compress_psnr
 * or the dense path's recon).  Q = L S, L = 2 mx my / (mx^2 + my^2), S = 2 s_xy / (s_x^2 + s_y^2);
 * reading R16: a 0/0 factor (denominator <= 1e-12 pixel^2) is 1.  x sums exact (int), y in fp64.
 *   x   [n][h][x_pitch] uint8;  y  [n][h][y_pitch bytes] float (4-byte aligned);
 *   uqi device double[n], overwritten.  n <= 65535.
 */
adct_status adct_uqi(const uint8_t* x, int64_t n, int64_t h, int64_t w, int64_t x_pitch, int64_t x_img_stride,
                     const float* y, int64_t y_pitch, int64_t y_img_stride, double* uqi, adct_stream_t stream);

/*
 * Parseval sweep: one read of the images yields the SSE of every triangular r.
 * Since C is orthogonal, the zonal error of a block equals its discarded orthonormal
 * energy: 576^2 SSE(r) = 576 sum_{zz >= r} W Y^2.  adct_diag_energy writes, per image, the exact
 * energies E[i][s] = sum over blocks of sum_{k+l=s} W_kl Y_kl^2, s = 0..14, and in entry 15 the
 * block energy E[i][15] = sum_all W Y^2 = 576 sum x^2 (P9 at r = 64; computed from the pixels)
 * (energy: device uint64[n][16], overwritten).  adct_diag_energy_prefix computes only the
 * anti-diagonals a sweep up to r_max needs (r_max <= 36: s = 0..7, the forward pruned to those 36
 * positions; otherwise all): entries it does not compute hold UINT64_MAX; EINVAL unless
 * 1 <= r_max <= 64.  adct_sweep_psnr turns either into SSE(r_s) = (E[15] - sum_{s' <= s} E[s']) / 576
 * and PSNR for every r that ends on a full anti-diagonal, r in {1,3,6,10,15,21,28,36,43,49,54,58,
 * 61,63,64} (host int r_list[n_r], n_r <= 16; other r -> ADCT_EINVAL): sse / psnr device
 * double[n_r][n], NaN where a needed entry is UINT64_MAX.  No inverse transform is computed: this
 * is a separate mode, not the fwd+zonal+inv path.
 */
adct_status adct_diag_energy(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                             int64_t img_stride, uint64_t* energy, adct_stream_t stream);
adct_status adct_diag_energy_prefix(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                                    int64_t img_stride, int r_max, uint64_t* energy, adct_stream_t stream);
adct_status adct_sweep_psnr(const uint64_t* energy, int64_t n, int64_t pixels, const int* r_list, int n_r,
                            double* sse, double* psnr, adct_stream_t stream);

/* HOST helper: the library's own 8x8 matrix for t (ADCT_T_PROPOSED..ADCT_T_COARSE, ADCT_T_CEIL),
 * row-major. */
adct_status adct_transform_matrix(adct_transform_t t, double* out);

/*
 * adct_quant_reciprocals — HOST helper, no device work: the 64 per-position fp32 constants c'
 * the QUANT kernels use (c' = smallest fp32 strictly above 1/(q sqrt(d_k d_l)), raster order
 * k*8+l), so that the quantiser decision round-to-nearest(Y c') can be audited on the CPU.
 *   c_out  host float[64].  ADCT_EINVAL if q <= 0, NaN or inf, or c_out is NULL.
 */
adct_status adct_quant_reciprocals(float q, float* c_out);

/* Human-readable status; static storage. */
const char* adct_status_string(adct_status s);
/* cudaError_t of the last ADCT_ECUDA on this thread (0 if none). */
int adct_last_cuda_error(void);
/* Library version (major * 10000 + minor * 100 + patch). */
int adct_version(void);
/* Number of kernel launches this library enqueued on this thread (bench instrumentation). */
int64_t adct_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* ADCT_H */
