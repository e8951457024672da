// adct_kernels.cuh — sm_100a kernel templates behind the C ABI (include/adct.h) for the arXiv 1402.6034
// hot path: blockwise 8x8 T X T^T with the 22-addition butterfly, S folded into the zonal /
// quantisation step, inverse with C^T, per-image SSE -> PSNR.  See DESIGN.md §5 for the
// data layout and the roofline of each kernel.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "adct_device.cuh"

#include <cuda_fp16.h>

#include <cuda/std/array>

namespace adct {

enum { MODE_ZONAL = 0, MODE_QUANT = 1 };
enum { OUT_I16 = 0, OUT_I32 = 1, OUT_F32 = 2 };
enum { REC_NONE = 0, REC_F32 = 1, REC_U8 = 2 };

// weight class of position (k, l): d_k d_l in {64, 48, 32, 36, 24, 16} -> 0..5
constexpr int wclass(int k, int l) {
  const int dd = dval(k) * dval(l);
  return dd == 64 ? 0 : dd == 48 ? 1 : dd == 32 ? 2 : dd == 36 ? 3 : dd == 24 ? 4 : 5;
}

struct Tables {
  float wc[8];   // ZONAL compile-time r: W per weight class (loop-invariant, uniform registers)
  float cc[8];   // ZONAL compile-time r: -KF * W per weight class
  float2 w[64];  // ZONAL: (W, W); QUANT: q / sqrt(d_k d_l); INVERSE: per-coef scale — 0 where masked
  float2 c[64];  // ZONAL: (-KF W, -KF W) [masked: 0]; QUANT: (c', c') quantiser reciprocal
  uint32_t keep[64];  // INVERSE: all ones where the zonal mask keeps the coefficient, else 0
  float sq[8];   // QUANT residual form: 1 / (q sqrt dd) per weight class as hi + lo fp32 pair
  float sql[8];
  float qscale;  // QUANT residual form: SSE = (q / 8)^2 * sum of the weighted inverse's squares
  float2 pm1;    // (1, -1): the uniform multiplicand pair of the one-instruction butterflies (inv8s)
  float2 pmr;    // (-1, 1): the swapped butterfly (sum in .y), inv8p's register-bank planning
  float2 ps2;    // (sqrt 2, -sqrt 2), (2 / sqrt 3, -2 / sqrt 3): the quantiser's weighted butterflies
  float2 pro;
};

// Deterministic per-image sums ("identical to sequential execution"; SURVEY §7 hard part 5):
// every LANE's partial of every TILE (a fixed-order fp32 sum of that tile's squared errors, which
// depends on nothing but the tile's pixels) is rounded once to the fixed-point grid 2^-k in pixel^2
// units and summed from there in 64-bit integers (per-lane accumulator, warp shuffle reduction,
// integer atomic per image).  Integer addition is associative, so the per-image total is
// bit-identical whatever the grid, the warp that processed a tile, the arrival order of the warps,
// the stream or the sharding of images across launches or ranks.  k is chosen per call on the host
// (fx_exponent in adct_api.cu) so that the largest possible per-image total stays below 2^61;
// k_fx_to_f64 converts the buffer in place afterwards (sse = total * 2^-k).  Rounding: at most
// 2^-(k+1) per (tile, lane), e.g. 0.016 pixel^2 over a whole 4096^2 image (SSE ~ 1e7 .. 1e9).
__device__ __forceinline__ long long fx_lane(float2 e2, float s) { return __float2ll_rn((e2.x + e2.y) * s); }
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void fx_flush(double* dst, long long v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(dst), (unsigned long long)v);
}
// a double partial (dense comparators, UQI): rounded once to the grid (the partial's own
// decomposition is fixed by the geometry: one 16 x 256 tile / one 32 x 32 window block)
__device__ __forceinline__ long long fx_of(double v, double scale) { return __double2ll_rn(v * scale); }

struct CompressParams {
  TileGeo geo;
  double fx_scale;     // 2^k: fixed-point scale of the deterministic per-image SSE (fx_lane / fx_flush)
  int64_t tiles;
  int cshift;  // log2 tiles per scheduling chunk
  int h, w;
  double* sse;
  uint8_t* recon;
  int64_t recon_pitch, recon_img_stride;
  int64_t sse_stride;  // multi-r kernel: distance between the per-r SSE rows (doubles)
  int rowmap[8];       // multi-r kernel: output row of the k-th r of the compiled set
  uint32_t h16magic;   // 0x64646464 from the host: a register operand, so the PRMT selector of the
                       // f16 pixel pairs stays an immediate (no per-PRMT selector materialisation)
  unsigned long long* sse576;  // k_compress_exact: exact per-image sum of (576 x - R)^2
  Tables tab;
};

struct ForwardParams {
  TileGeo geo;
  int64_t tiles;
  int cshift;
  int h, w;
  uint8_t* coef;
  int64_t coef_pitch, coef_img_stride;
  int masked;        // r < 64
  uint32_t m16[32];  // I16: AND-mask per coefficient pair (row k, pair m) -> index k*4+m
  uint64_t keep_raster;  // bit k*8+l: coefficient (k, l) kept
  float sc[64];      // F32: fp32(1/sqrt(d_i d_j)), 0 where masked
};

struct InverseParams {
  TileGeo geo;
  int64_t tiles;
  int cshift;  // TMA (int16) path: log2 tiles per scheduling chunk
  int h, w;
  const uint8_t* coef;
  int64_t coef_pitch, coef_img_stride;
  uint8_t* dst;
  int64_t dst_pitch, dst_img_stride;
  Tables tab;  // w[k]: multiplier applied to the loaded coefficient (W or 1/sqrt(dd)), 0 if masked
};

// ------------------------------------------------------------------------------------------
// Reconstruction store for row I (8 pixels of block A and of block B) — masked to the image.
// ------------------------------------------------------------------------------------------
// u8 reconstruction of one output row of both blocks, x[n] = (A, B) pair of pixel n.
// S576: u8 = clamp(round_half_away(R / 576)) = clamp(floor((R + 288.5) / 576)) for integer R
// (never within 8.7e-4 of an integer, so the fp32 product is floored exactly); else clamp(floor(x^ + 0.5)).
// Fast form (SAFE = false): one FADD2 + one round-toward-zero FFMA2 with the magic 2^23 + 512 per pixel
// pair puts floor(y) + 512 in the low 16 bits; two halves pack into one word, clamp to [512, 767] with
// VIMNMX.U16x2, and the low bytes are floor(y) clamped to [0, 255].  The magic holds only for
// floor(y) in [-512, 65023]: the fused zonal compress uses it because its R is proven inside
// [-182325, 329205] (y in [-316, 572], tools/exactness_bounds.py).
// SAFE = true (quantiser reconstruction, inverse from arbitrary coefficient planes): y is first
// saturated to [0, 256] / 256 by one scalar FFMA.SAT per value (NaN -> 0), z = sat((y + 0.5) / 256),
// then floor(256 z) + 512 by the same round-toward-zero FFMA2 — every input clamps correctly.
// For S576 the scaled sum RN(R / 147456 + 288.5 / 147456) is within 3e-5 (in pixel units) of
// (R + 288.5) / 576 for every R that does not saturate, far inside the 8.7e-4 margin.
// u8 rounding kinds: exact-integer R = 576 x^ (fast magic / saturating), real R = 576 x^ (from an f32
// coefficient plane: round_half_away(R / 576) with no integer offset), real x^ (quantiser).
enum { U8_FAST576 = 0, U8_SAFE576 = 1, U8_SAFE576R = 2, U8_SAFEX = 3 };
template <int U8K>
__device__ __forceinline__ void u8_rows(const float2 (&x)[8], uint2& ra, uint2& rb) {
  constexpr bool SAFE = U8K == U8_SAFE576 || U8K == U8_SAFE576R || U8K == U8_SAFEX;
  constexpr bool S576 = U8K == U8_FAST576 || U8K == U8_SAFE576 || U8K == U8_SAFE576R;
  uint32_t ta[8], tb[8];
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    float2 t;
    if constexpr (SAFE) {
      constexpr float c1 = S576 ? (float)(1.0 / 147456.0) : 0.00390625f;
      constexpr float c2 = U8K == U8_SAFE576 ? (float)(288.5 / 147456.0) : 0.001953125f;
      float za, zb;
      asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(za) : "f"(x[n].x), "f"(c1), "f"(c2));
      asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(zb) : "f"(x[n].y), "f"(c1), "f"(c2));
      const float2 z = make_float2(za, zb);
      unsigned long long d;
      asm("fma.rz.f32x2 %0, %1, %2, %3;" : "=l"(d)
          : "l"(*reinterpret_cast<const unsigned long long*>(&z)), "l"(0x4380000043800000ull),
            "l"(0x4B0002004B000200ull));
      t = *reinterpret_cast<float2*>(&d);
    } else {
      static_assert(U8K == U8_FAST576, "fast form: exact-integer R only");
      const float2 sft = f2add(x[n], f2(288.5f));  // exact: R is an integer below 2^19
      unsigned long long d;
      asm("fma.rz.f32x2 %0, %1, %2, %3;" : "=l"(d)
          : "l"(*reinterpret_cast<const unsigned long long*>(&sft)), "l"(0x3AE38E393AE38E39ull),
            "l"(0x4B0002004B000200ull));
      t = *reinterpret_cast<float2*>(&d);
    }
    ta[n] = __float_as_uint(t.x);
    tb[n] = __float_as_uint(t.y);
  }
  uint32_t pa[4], pb[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    pa[q] = __byte_perm(ta[2 * q], ta[2 * q + 1], 0x5410);
    pb[q] = __byte_perm(tb[2 * q], tb[2 * q + 1], 0x5410);
    asm("max.u16x2 %0, %0, %1;" : "+r"(pa[q]) : "r"(0x02000200u));
    asm("min.u16x2 %0, %0, %1;" : "+r"(pa[q]) : "r"(0x02FF02FFu));
    asm("max.u16x2 %0, %0, %1;" : "+r"(pb[q]) : "r"(0x02000200u));
    asm("min.u16x2 %0, %0, %1;" : "+r"(pb[q]) : "r"(0x02FF02FFu));
  }
  ra = make_uint2(__byte_perm(pa[0], pa[1], 0x6420), __byte_perm(pa[2], pa[3], 0x6420));
  rb = make_uint2(__byte_perm(pb[0], pb[1], 0x6420), __byte_perm(pb[2], pb[3], 0x6420));
}

template <int RECON, bool S576, int U8K>
__device__ __forceinline__ void store_recon_row(uint8_t* base, int64_t pitch, int h, int w, int row_a,
                                                int col, const float2 (&x)[8]) {
  // S576: x[n] = (R_A[n], R_B[n]) with R = 576 x^ exactly (integers in fp32); else x[n] = x^ itself
  if (col >= w) return;
  if (RECON == REC_U8 && row_a >= h) return;
  const int rows[2] = {row_a, row_a + 8};
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    if (RECON == REC_U8 || rows[b] >= h) continue;
    uint8_t* p = base + (int64_t)rows[b] * pitch;
    if constexpr (RECON == REC_F32) {
      float v[8];
#pragma unroll
      for (int n = 0; n < 8; ++n) v[n] = S576 ? (b ? x[n].y : x[n].x) * (1.0f / 576.0f) : (b ? x[n].y : x[n].x);
      float4* q = reinterpret_cast<float4*>(p + (int64_t)col * 4);
      q[0] = make_float4(v[0], v[1], v[2], v[3]);
      q[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
  if constexpr (RECON == REC_U8) {
    uint2 ra, rb;
    u8_rows<U8K>(x, ra, rb);
    *reinterpret_cast<uint2*>(base + (int64_t)row_a * pitch + col) = ra;
    if (row_a + 8 < h) *reinterpret_cast<uint2*>(base + (int64_t)(row_a + 8) * pitch + col) = rb;
  }
}

// The same two output rows into a warp-private shared-memory staging tile laid out as the 16 x 256
// box of a TMA bulk-tensor store (f32: 1 KiB per row, u8: 256 B per row).
template <int RECON, bool S576, int U8K>
__device__ __forceinline__ void stage_recon_row(uint8_t* buf, int row_a, int lane, const float2 (&x)[8]) {
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    const int row = row_a + 8 * b;
    if constexpr (RECON == REC_F32) {
      float v[8];
#pragma unroll
      for (int n = 0; n < 8; ++n) v[n] = S576 ? (b ? x[n].y : x[n].x) * (1.0f / 576.0f) : (b ? x[n].y : x[n].x);
      float4* q = reinterpret_cast<float4*>(buf + row * (4 * TILE_W) + lane * 32);
      q[0] = make_float4(v[0], v[1], v[2], v[3]);
      q[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
  if constexpr (RECON == REC_U8) {
    uint2 ra, rb;
    u8_rows<U8K>(x, ra, rb);
    *reinterpret_cast<uint2*>(buf + row_a * TILE_W + lane * 8) = ra;
    *reinterpret_cast<uint2*>(buf + (row_a + 8) * TILE_W + lane * 8) = rb;
  }
}
constexpr int recon_stage_bytes(int RECON) { return RECON == REC_F32 ? 4 * TILE_BYTES : TILE_BYTES; }

// ------------------------------------------------------------------------------------------
// Fused compress path, split in two halves so that a warp can overlap the ALU-heavy forward of
// tile j+1 (SWAR IADD3/PRMT) with the FMA-heavy inverse + error of tile j (FADD2/FFMA2) in one
// basic block: ptxas interleaves the two independent streams and both pipes stay busy.
// ------------------------------------------------------------------------------------------

// Forward half: packed SWAR coefficients Y (bias 0x80008000) of the two blocks of this lane.
template <int R, int MODE, bool MIRB = false>
__device__ __forceinline__ void compress_fwd(const uint8_t* tile, int lane, uint32_t (&Y)[8][8]) {
  constexpr int RF = R;  // forward pruning level (RT: runtime mask, all positions live)
  uint32_t P[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
    pack_rows_t<MIRB>(lds64(tile + i * TILE_W + lane * 8), lds64(tile + (i + 8) * TILE_W + lane * 8), P[i]);
  fwd2d<BIAS2, RF>(P, Y);
}
// ... and the row pass H of the columns in SKIP (their column pass is skipped)
template <int R, int SKIP, bool MIRB = false>
__device__ __forceinline__ void compress_fwd_h(const uint8_t* tile, int lane, uint32_t (&Y)[8][8], uint32_t (&H)[8][8]) {
  uint32_t P[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
    pack_rows_t<MIRB>(lds64(tile + i * TILE_W + lane * 8), lds64(tile + (i + 8) * TILE_W + lane * 8), P[i]);
  fwd2d<BIAS2, R, SKIP>(P, Y, H);
}

// Inverse half: zonal weights / quantiser, inverse with C^T, error against the staged pixels.
// Returns this lane's partial sum of squared errors (576 units for ZONAL) as an fp32 pair.
// F16 (compile-time r, zonal, SSE only): the first F16 output rows take their pixels through the
// f16 magic — one PRMT makes the f16 pair (1024 + x_n, 1024 + x_{n+1}) of two pixels of a block —
// and each pixel's error is ONE mixed-precision FMA (PTX fma.rn.f32.f16, SASS FHFMA: f16 x f16 +
// f32 -> f32, full rate on the FMA pipe, the f16 half selected in the operand):
// e = R' - 576 (1024 + x) with R' = R + 589824 injected at the DC weight (T's first row is all
// ones, so a constant added to V_00 shifts every output by the same amount; |R'| < 2^24 stays
// exact, tools/exactness_bounds.py) — the product 576 (1024 + x) is exact inside the FMA.  Per
// pixel pair: 1 PRMT + 2 FHFMA (vs 2 PRMT + FFMA2 + FADD2 on the f32 route): -1 ALU and -2
// FMA-pipe cycles.  The other rows keep the f32 magic.
constexpr float DC_BIAS16 = 589824.0f;  // 576 * 1024
// 0xE080 = f16(-576), 0x6080 = f16(+576): the sign follows the typed row output (FV<neg> stores -R')
template <bool HI, bool NEG>
__device__ __forceinline__ float fhfma576(uint32_t h2, float c) {
  float d;
  if constexpr (HI)
    asm("{.reg .f16 a, b; mov.b32 {_, a}, %1; mov.b16 b, %3; fma.rn.f32.f16 %0, a, b, %2;}"
        : "=f"(d) : "r"(h2), "f"(c), "n"(NEG ? 0x6080 : 0xE080));
  else
    asm("{.reg .f16 a, b; mov.b32 {a, _}, %1; mov.b16 b, %3; fma.rn.f32.f16 %0, a, b, %2;}"
        : "=f"(d) : "r"(h2), "f"(c), "n"(NEG ? 0x6080 : 0xE080));
  return d;
}
// e for pixel N of row (A, B): R' -/+ 576 (1024 + x), exact
template <int N, bool NEG>
__device__ __forceinline__ float2 err_fh(uint32_t ha, uint32_t hb, float2 v) {
  return make_float2(fhfma576<(N & 1) != 0, NEG>(ha, v.x), fhfma576<(N & 1) != 0, NEG>(hb, v.y));
}
template <int N> __device__ __forceinline__ float2 err_fh(uint32_t ha, uint32_t hb, FV<false> r) {
  return err_fh<N, false>(ha, hb, r.v);
}
template <int N> __device__ __forceinline__ float2 err_fh(uint32_t ha, uint32_t hb, FV<true> r) {
  return err_fh<N, true>(ha, hb, r.v);
}

// Scalar-per-block inverse (inverse2d_s, adct_device.cuh) -> the (block A, block B) view the error
// callbacks use: output n of both blocks as one typed value (no register pair is formed for the
// scalar consumers, FHFMA / FFMA).
// Inverse flavour per kernel (template parameter SM): 0 = f32x2 FADD2 over the (A, B) block pair,
// 1 = per-block scalar one-instruction butterflies (inv8s), 2 = the same with a register-bank plan
// (inv8p).  Measured on B200 (profiles/r02_variants_inverse_flavour.txt, 1024 C5 images): SM = 1 wins
// for the direct form at small r (r = 6: 0.75 -> 0.85 of HBM, r = 10: 0.63 -> 0.69) and for the
// residual form (r = 28: 0.57 -> 0.60, r = 36: 0.61 -> 0.66); the grouped mid-r kernels (11 <= r < 24)
// and C4's quantiser keep SM = 0; the bank plan (SM = 2) did not pay (ptxas re-assigns registers).
#ifndef ADCT_SINV
#define ADCT_SINV -1  // -1: the measured per-kernel choice (sinv_mode); 0 / 1 / 2 force one flavour
#endif
template <bool N> __device__ __forceinline__ FV<N> join_ab(SV<N> a, SV<N> b) { return {make_float2(a.v, b.v)}; }
__device__ __forceinline__ Z0 join_ab(Z0, Z0) { return {}; }
template <class RA, class RB> __device__ __forceinline__ auto join_rows(const RA& ra, const RB& rb) {
  using cuda::std::get;
  return cuda::std::make_tuple(join_ab(get<0>(ra), get<0>(rb)), join_ab(get<1>(ra), get<1>(rb)),
                               join_ab(get<2>(ra), get<2>(rb)), join_ab(get<3>(ra), get<3>(rb)),
                               join_ab(get<4>(ra), get<4>(rb)), join_ab(get<5>(ra), get<5>(rb)),
                               join_ab(get<6>(ra), get<6>(rb)), join_ab(get<7>(ra), get<7>(rb)));
}
// acc += (a, b)^2 for outputs n, 7 - n of ONE block (they leave one butterfly as a register pair)
__device__ __forceinline__ float2 sq2(Z0, Z0, float2 acc) { return acc; }
template <bool NA> __device__ __forceinline__ float2 sq2(SV<NA> a, Z0, float2 acc) {
  return make_float2(fmaf(a.v, a.v, acc.x), acc.y);
}
template <bool NB> __device__ __forceinline__ float2 sq2(Z0, SV<NB> b, float2 acc) {
  return make_float2(acc.x, fmaf(b.v, b.v, acc.y));
}
template <bool NA, bool NB> __device__ __forceinline__ float2 sq2(SV<NA> a, SV<NB> b, float2 acc) {
  const float2 v = make_float2(a.v, b.v);
  return f2fma(v, v, acc);
}

// block BLK's biased float 2^23 + 2^15 + Y of a packed coefficient (the halves of biased_pair)
template <int BLK> __device__ __forceinline__ float bpf(uint32_t Pb) {
  return __uint_as_float(__byte_perm(Pb, 0x4B000000u, BLK ? 0x7632 : 0x7610));
}
// W . Y of the kept set KS (compile-time mask) into per-block scalar planes, the column partners
// (0,4), (6,2), (1,3), (7,5) converted as one register pair each (inv8p's input parity pattern);
// partners share the weight class.  dc adds a constant to coefficient (0, 0) (the f16 route's bias).
template <int KS>
__device__ __forceinline__ void convert_planned(const uint32_t (&Y)[8][8], const CompressParams& p, float dc,
                                                float (&VS)[2][64]) {
  static_for<64>([&](auto KLc) {
    constexpr int kl = decltype(KLc)::value, k = kl / 8, l = kl % 8, k2 = pair_partner(k);
    constexpr int c = wclass(k, l);
    static_assert(wclass(k, l) == wclass(k2, l), "partners share the weight class");
    if constexpr (kept(KS, k, l) && pair_lead(k) && kept(KS, k2, l)) {
      const float cc = p.tab.cc[c];
      const float c0 = kl == 0 ? cc + dc : cc;
      static_for<2>([&](auto Bc) {
        constexpr int B = decltype(Bc)::value;
        const float2 v = f2fma(make_float2(bpf<B>(Y[k][l]), bpf<B>(Y[k2][l])), f2(p.tab.wc[c]), make_float2(c0, cc));
        VS[B][k * 8 + l] = v.x;
        VS[B][k2 * 8 + l] = v.y;
      });
    } else if constexpr (kept(KS, k, l) && !kept(KS, k2, l)) {  // lone member: a scalar FFMA
      const float cc = kl == 0 ? p.tab.cc[c] + dc : p.tab.cc[c];
      VS[0][kl] = fmaf(bpf<0>(Y[k][l]), p.tab.wc[c], cc);
      VS[1][kl] = fmaf(bpf<1>(Y[k][l]), p.tab.wc[c], cc);
    }
  });
}

template <int R, int MODE, int RECON, int F16 = 0, bool GROUPED = false, bool STAGE = false, bool MIRB = false,
          int SM = 0>
__device__ __forceinline__ float2 compress_inv(const uint32_t (&Y)[8][8], const uint8_t* tile, int lane,
                                               const CompressParams& p, int img, int ty, int tx,
                                               uint8_t* sbuf = nullptr) {
  constexpr int RF = R;
  static_assert(!MIRB || RECON == REC_NONE, "mirrored block B: SSE only (the reconstruction would be mirrored)");
  static_assert(F16 == 0 || (MODE == MODE_ZONAL && RECON == REC_NONE && RF < RT), "f16 error route: zonal SSE only");
  float2 V[64];
  static_for<64>([&](auto KLc) {
    constexpr int kl = decltype(KLc)::value, k = kl / 8, l = kl % 8;
    if constexpr (kept(RF, k, l)) {
      if constexpr (MODE == MODE_ZONAL && RF < RT) {
        // scalar weight / offset broadcast to both lanes from 12 loop-invariant class constants:
        // an FFMA2 that reads three distinct register pairs issues at 2/3 rate on B200 (tools/microbench/ffma2_forms.cu)
        constexpr int c = wclass(k, l);
        const float cc = (F16 > 0 && kl == 0) ? p.tab.cc[c] + DC_BIAS16 : p.tab.cc[c];
        V[kl] = f2fma(biased_pair(Y[k][l]), f2(p.tab.wc[c]), f2(cc));  // W . M . Y (+ bias), exact
      } else if constexpr (MODE == MODE_ZONAL) {
        V[kl] = f2fma(biased_pair(Y[k][l]), f2(p.tab.w[kl].x), f2(p.tab.c[kl].x));  // runtime mask in w
      } else {
        const float2 y = f2add(biased_pair(Y[k][l]), f2(-KF));          // Y, exact
        // 1.5*2^23 + RN(Y c'): c' lies strictly above 1/(q sqrt dd), so exact ties of Z/q round
        // away from zero and no product Y c' is itself a tie (reading R10)
        if constexpr (RF < RT) {  // compile-time mask: per-class scalars (q / sqrt dd, c')
          constexpr int c = wclass(k, l);
          const float2 t = f2fma(y, f2(p.tab.cc[c]), f2(12582912.0f));
          V[kl] = __fmul2_rn(f2add(t, f2(-12582912.0f)), f2(p.tab.wc[c]));
        } else {
          const float2 t = f2fma(y, p.tab.c[kl], f2(12582912.0f));
          V[kl] = __fmul2_rn(f2add(t, f2(-12582912.0f)), p.tab.w[kl]);   // q k / sqrt(dd) (M folded)
        }
      }
    }
  });

  float2 acc[8];  // one accumulator chain per column: 8 short FFMA2 chains instead of one long one
#pragma unroll
  for (int n = 0; n < 8; ++n) acc[n] = f2(0.f);
  const int col = tx * TILE_W + lane * 8;
  uint8_t* rbase = nullptr;
  if constexpr (RECON != REC_NONE) rbase = p.recon + (int64_t)img * p.recon_img_stride;
  auto err_row = [&](auto Ic, auto row) {
    constexpr int I = decltype(Ic)::value;
    using cuda::std::get;
    const uint2 wa = lds64_reload(tile + I * TILE_W + lane * 8);
    const uint2 wb = lds64_reload(tile + (I + 8) * TILE_W + lane * 8);
    [[maybe_unused]] float2 xr[8];  // reconstruction row (RECON kernels only)
    static_for<8>([&](auto Nc) {
      constexpr int N = decltype(Nc)::value;
      if constexpr (I < F16) {
        // f16 pairs (1024 + x_n, 1024 + x_{n+1}) of blocks A and B, one PRMT each per two pixels
        // (MIRB: B's output column n is its pixel 7 - n: the pair (x_{7-n}, x_{6-n}))
        constexpr uint32_t sel = ((N >> 1) & 1) ? 0x4342u : 0x4140u;
        constexpr uint32_t selb = MIRB ? (((N >> 1) & 1) ? 0x4041u : 0x4243u) : sel;
        const uint32_t ha = __byte_perm(N < 4 ? wa.x : wa.y, p.h16magic, sel);
        const uint32_t hb = __byte_perm((N < 4) != MIRB ? wb.x : wb.y, p.h16magic, selb);
        const float2 e = err_fh<N>(ha, hb, get<N>(row));  // R' - 576 (1024 + x) = R - 576 x, exact
        acc[N] = f2fma(e, e, acc[N]);
      } else {
        // ZONAL: 576 x - R, exact integers; QUANT: x - x^ (fp32, irrational weights)
        constexpr int NB = MIRB ? 7 - N : N;  // block B's pixel in output column N
        const float2 y = (MODE == MODE_ZONAL)
                             ? px576b2<(F16 > 0)>(N < 4 ? wa.x : wa.y, NB < 4 ? wb.x : wb.y, N & 3, NB & 3)
                             : px1(N < 4 ? wa.x : wa.y, N < 4 ? wb.x : wb.y, N & 3);
        const float2 e = rsub(y, get<N>(row));
        acc[N] = f2fma(e, e, acc[N]);
        if constexpr (RECON != REC_NONE) xr[N] = val(get<N>(row));
      }
    });
    if constexpr (RECON != REC_NONE && STAGE) stage_recon_row<RECON, (MODE == MODE_ZONAL), (MODE == MODE_ZONAL ? U8_FAST576 : U8_SAFEX)>(sbuf, I, lane, xr);
    else if constexpr (RECON != REC_NONE)
      store_recon_row<RECON, (MODE == MODE_ZONAL), (MODE == MODE_ZONAL ? U8_FAST576 : U8_SAFEX)>(rbase, p.recon_pitch, p.h, p.w, ty * TILE_H + I, col, xr);
  };
  if constexpr (SM == 4 && MODE == MODE_ZONAL && RECON == REC_NONE && RF < RT && F16 == 8) {
    // one block at a time in a run-time loop (half the live floats of the (A, B) forms): per-block
    // scalar plane, one-instruction butterflies, each pixel's error through FHFMA, squares of the
    // (n, 7 - n) output pairs of one block
#pragma unroll 1
    for (int blk = 0; blk < 2; ++blk) {
      const uint32_t csel = blk ? 0x7632u : 0x7610u;
      float2 V1[64];
      static_for<64>([&](auto KLc) {
        constexpr int kl = decltype(KLc)::value, k = kl / 8, l = kl % 8;
        if constexpr (kept(RF, k, l)) {
          constexpr int c = wclass(k, l);
          const float cc = kl == 0 ? p.tab.cc[c] + DC_BIAS16 : p.tab.cc[c];
          V1[kl] = make_float2(fmaf(__uint_as_float(__byte_perm(Y[k][l], 0x4B000000u, csel)), p.tab.wc[c], cc), 0.f);
        }
      });
      const bool mir = MIRB && blk;  // block B column-mirrored: output column N is its pixel 7 - N
      inverse2d_s1<RF>(V1, p.tab.pm1, [&](auto Ic, const auto& ra) {
        constexpr int I = decltype(Ic)::value;
        using cuda::std::get;
        const uint2 w = lds64_reload(tile + (I + 8 * blk) * TILE_W + lane * 8);
        auto err = [&](auto Mc) {  // R' - 576 (1024 + x) = R - 576 x for output column M, exact
          constexpr int M = decltype(Mc)::value;
          constexpr uint32_t sel = ((M >> 1) & 1) ? 0x4342u : 0x4140u;
          constexpr uint32_t selm = ((M >> 1) & 1) ? 0x4041u : 0x4243u;
          const uint32_t h = __byte_perm(((M < 4) != mir) ? w.x : w.y, p.h16magic, mir ? selm : sel);
          const auto r = get<M>(ra);
          return fhfma576<(M & 1) != 0, cuda::std::decay_t<decltype(r)>::neg>(h, r.v);
        };
        static_for<4>([&](auto Nc) {
          constexpr int N = decltype(Nc)::value;
          const float2 e = make_float2(err(cuda::std::integral_constant<int, N>{}),
                                       err(cuda::std::integral_constant<int, 7 - N>{}));
          acc[N] = f2fma(e, e, acc[N]);
        });
      });
    }
  } else if constexpr (SM == 2 && MODE == MODE_ZONAL && RF < RT && !GROUPED) {
    // bank-planned scalar inverse (inv8p) on per-block planes converted as register pairs
    float VS[2][64], UHS[2][8][8];
    convert_planned<RF>(Y, p, F16 > 0 ? DC_BIAS16 : 0.f, VS);
    auto err_row_s = [&](auto Ic, const auto& ra, const auto& rb) { err_row(Ic, join_rows(ra, rb)); };
    inverse2d_p<RF>(VS, UHS, p.tab.pm1, p.tab.pmr, err_row_s);
  } else if constexpr (SM == 3) {  // f32x2 column pass, scalar-butterfly row pass
    auto err_row_s = [&](auto Ic, const auto& ra, const auto& rb) { err_row(Ic, join_rows(ra, rb)); };
    if constexpr (GROUPED) inverse2d_hyb_grouped<RF>(V, p.tab.pm1, err_row_s);
    else inverse2d_hyb<RF>(V, p.tab.pm1, err_row_s);
  } else if constexpr (SM != 0) {
    auto err_row_s = [&](auto Ic, const auto& ra, const auto& rb) { err_row(Ic, join_rows(ra, rb)); };
    float2 UH[8][8];  // unused (no injected columns in the direct form)
    if constexpr (GROUPED) inverse2d_s_grouped<RF>(V, p.tab.pm1, err_row_s);
    else inverse2d_s<RF>(V, UH, p.tab.pm1, err_row_s);
  } else {
    if constexpr (GROUPED) inverse2d_grouped<RF>(V, err_row);
    else inverse2d<RF>(V, err_row);
  }
  const float2 s01 = f2add(acc[0], acc[1]), s23 = f2add(acc[2], acc[3]);
  const float2 s45 = f2add(acc[4], acc[5]), s67 = f2add(acc[6], acc[7]);
  return f2add(f2add(s01, s23), f2add(s45, s67));
}

// Residual form of the zonal error (compile-time r, SSE only).  C = D C0 is orthogonal, so
// C0^T (W . Y) C0 = 576 x for every block (r = 64 is lossless, pin P8) and, by linearity,
//     576 x - R_r = C0^T (W . (1 - M_r) . Y) C0,
// i.e. the reconstruction error of the zonal step is the same inverse butterfly applied to the
// coefficients the mask discards.  Every node is an integer below 2^24 (tools/exactness_bounds.py),
// so this equals the direct form bit for bit; it needs no pixel re-read and no 576 x, and for
// large r the discarded set is the smaller one.  Returns the lane's sum of e^2 (576 units).
template <int R, bool GROUPED = false, int SM = 0>
__device__ __forceinline__ float2 compress_resid(const uint32_t (&Y)[8][8], const CompressParams& p) {
  constexpr int RM = RESID + R;
  float2 V[64];
  static_for<64>([&](auto KLc) {
    constexpr int kl = decltype(KLc)::value, k = kl / 8, l = kl % 8;
    if constexpr (kept(RM, k, l)) {
      constexpr int c = wclass(k, l);
      V[kl] = f2fma(biased_pair(Y[k][l]), f2(p.tab.wc[c]), f2(p.tab.cc[c]));  // W . (1 - M) . Y, exact
    }
  });
  float2 acc[8];
#pragma unroll
  for (int n = 0; n < 8; ++n) acc[n] = f2(0.f);
  auto sq_row = [&](auto Ic, auto row) {
    using cuda::std::get;
    static_for<8>([&](auto Nc) {
      constexpr int N = decltype(Nc)::value;
      acc[N] = sqacc(get<N>(row), acc[N]);
    });
  };
  // per block: outputs n and 7 - n leave one butterfly as a register pair -> one FFMA2 per pair
  auto sq_row_s = [&](auto Ic, const auto& ra, const auto& rb) {
    using cuda::std::get;
    static_for<4>([&](auto Nc) {
      constexpr int N = decltype(Nc)::value;
      acc[N] = sq2(get<N>(ra), get<7 - N>(ra), acc[N]);
      acc[4 + N] = sq2(get<N>(rb), get<7 - N>(rb), acc[4 + N]);
    });
  };
  if constexpr (SM == 4 && !GROUPED) {  // one block at a time in a run-time loop (see compress_inv)
#pragma unroll 1
    for (int blk = 0; blk < 2; ++blk) {
      const uint32_t csel = blk ? 0x7632u : 0x7610u;
      float2 V1[64];
      static_for<64>([&](auto KLc) {
        constexpr int kl = decltype(KLc)::value, k = kl / 8, l = kl % 8;
        if constexpr (kept(RM, k, l)) {
          constexpr int c = wclass(k, l);
          V1[kl] = make_float2(fmaf(__uint_as_float(__byte_perm(Y[k][l], 0x4B000000u, csel)), p.tab.wc[c], p.tab.cc[c]), 0.f);
        }
      });
      inverse2d_s1<RM>(V1, p.tab.pm1, [&](auto Ic, const auto& ra) {
        using cuda::std::get;
        static_for<4>([&](auto Nc) {
          constexpr int N = decltype(Nc)::value;
          acc[N] = sq2(get<N>(ra), get<7 - N>(ra), acc[N]);
        });
      });
    }
  } else if constexpr (SM == 2 && !GROUPED) {
    float VS[2][64], UHS[2][8][8];
    convert_planned<RM>(Y, p, 0.f, VS);
    inverse2d_p<RM>(VS, UHS, p.tab.pm1, p.tab.pmr, sq_row_s);
  } else if constexpr (SM == 3) {
    if constexpr (GROUPED) inverse2d_hyb_grouped<RM>(V, p.tab.pm1, sq_row_s);
    else inverse2d_hyb<RM>(V, p.tab.pm1, sq_row_s);
  } else if constexpr (SM != 0) {
    float2 UH[8][8];
    if constexpr (GROUPED) inverse2d_s_grouped<RM>(V, p.tab.pm1, sq_row_s);
    else inverse2d_s<RM>(V, UH, p.tab.pm1, sq_row_s);
  } else {
    if constexpr (GROUPED) inverse2d_grouped<RM>(V, sq_row);
    else inverse2d<RM>(V, sq_row);
  }
  const float2 s01 = f2add(acc[0], acc[1]), s23 = f2add(acc[2], acc[3]);
  const float2 s45 = f2add(acc[4], acc[5]), s67 = f2add(acc[6], acc[7]);
  return f2add(f2add(s01, s23), f2add(s45, s67));
}

// Residual form with the fully discarded columns injected from the row pass (inverse2d_hc):
// UH[L][i] = (576 / d_L) H[i][L], exact integers (< 2^18) — the same column-pass values as the
// coefficient route, so every later node (and the exactness proof) is unchanged.
#ifndef ADCT_RESID_HC
#define ADCT_RESID_HC 1
#endif
#ifndef ADCT_RESID_P2
#define ADCT_RESID_P2 1  // also inject the columns whose kept set is exactly {(0, L), (1, L)}
#endif
#ifndef ADCT_P2_LO
#define ADCT_P2_LO 27  // measured per r (profiles/r02_variants_partial_injection.txt): +2-6 % at
#endif                 // r = 27..35 (r = 28 +6 %), -3 % at r = 24 and -1 % at r = 36
#ifndef ADCT_P2_HI
#define ADCT_P2_HI 35
#endif
constexpr int resid_p2_mask(int R) {
  return (ADCT_RESID_P2 && R >= ADCT_P2_LO && R <= ADCT_P2_HI) ? p2col_mask(R) : 0;
}
#ifndef ADCT_RESID_PC
#define ADCT_RESID_PC 1  // also inject the columns whose only kept coefficient is (0, L) (pcol_mask)
#endif
template <int R, int SM = 0>
__device__ __forceinline__ float2 compress_resid_hc(const uint32_t (&Y)[8][8], const uint32_t (&H)[8][8],
                                                    const CompressParams& p) {
  constexpr int PC = ADCT_RESID_PC ? pcol_mask(R) : 0;
  constexpr int P2 = resid_p2_mask(R);
  constexpr int RM = RESID + R, HC = hcol_mask(R) | PC | P2;  // every injected column
  static_assert(PC == 0 || SM != 2, "the bank-planned flavour injects only fully discarded columns");
  float2 V[64];
  static_for<64>([&](auto KLc) {
    constexpr int kl = decltype(KLc)::value, k = kl / 8, l = kl % 8;
    if constexpr (kept(RM, k, l) && !((HC >> l) & 1)) {
      constexpr int c = wclass(k, l);
      V[kl] = f2fma(biased_pair(Y[k][l]), f2(p.tab.wc[c]), f2(p.tab.cc[c]));  // W . (1 - M) . Y, exact
    }
  });
  float2 UH[8][8];
  static_for<8>([&](auto Lc) {
    constexpr int L = decltype(Lc)::value;
    if constexpr ((P2 >> L) & 1) {
      // kept rows {0, 1}: W_0L (8 H - Y_0L) - T1[i] W_1L Y_1L, Y_1L = sum_i T1[i] H[i][L] (|.| <= 6120)
      const uint32_t y0 = ((H[0][L] + H[1][L]) + (H[2][L] + H[3][L])) + ((H[4][L] + H[5][L]) + (H[6][L] + H[7][L]));
      const uint32_t y1 = (H[0][L] + H[1][L] + H[2][L]) - (H[5][L] + H[6][L] + H[7][L]);
      const uint32_t off = BIAS2 - y0;
      constexpr float w0 = (float)(576 / (8 * dval(L))), w1 = (float)(576 / (6 * dval(L)));
      const float2 v1 = f2fma(biased_pair(y1 + BIAS2), f2(w1), f2(-KF * w1));
      static_for<8>([&](auto Ic) {
        constexpr int i = decltype(Ic)::value;
        const float2 u = f2fma(biased_pair((H[i][L] << 3) + off), f2(w0), f2(-KF * w0));
        UH[L][i] = i < 3 ? f2sub(u, v1) : i > 4 ? f2add(u, v1) : u;
      });
    } else if constexpr ((PC >> L) & 1) {
      // only (0, L) kept: the discarded rows' column inverse is (576 / d_L) H[:, L] - W_0L Y_0L =
      // (W_0L) (8 H[i][L] - Y_0L) with W_0L = 576 / (8 d_L) an integer and Y_0L = sum_i H[i][L]:
      // 8 H - Y_0L is an exact int16 SWAR lane (|.| <= 32640), one LEA per row, then the same
      // magic-exponent conversion as a fully injected column
      const uint32_t y0 = ((H[0][L] + H[1][L]) + (H[2][L] + H[3][L])) + ((H[4][L] + H[5][L]) + (H[6][L] + H[7][L]));
      const uint32_t off = BIAS2 - y0;
      constexpr float w0 = (float)(576 / (8 * dval(L)));
#pragma unroll
      for (int i = 0; i < 8; ++i)
        UH[L][i] = f2fma(biased_pair((H[i][L] << 3) + off), f2(w0), f2(-KF * w0));
    } else if constexpr ((HC >> L) & 1) {
      constexpr float wl = (float)(576 / dval(L));
#pragma unroll
      for (int i = 0; i < 8; ++i)  // + 0x80008000: both 16-bit lanes biased (the low lane's borrow cancels)
        UH[L][i] = f2fma(biased_pair(H[i][L] + BIAS2), f2(wl), f2(-KF * wl));
    }
  });
  float2 acc[8];
#pragma unroll
  for (int n = 0; n < 8; ++n) acc[n] = f2(0.f);
  if constexpr (SM != 0) {
    auto sq_row_s = [&](auto Ic, const auto& ra, const auto& rb) {
      using cuda::std::get;
      static_for<4>([&](auto Nc) {
        constexpr int N = decltype(Nc)::value;
        acc[N] = sq2(get<N>(ra), get<7 - N>(ra), acc[N]);
        acc[4 + N] = sq2(get<N>(rb), get<7 - N>(rb), acc[4 + N]);
      });
    };
    if constexpr (SM == 2) {
      float VS[2][64], UHS[2][8][8];
      convert_planned<RM & 0 ? 0 : (RM)>(Y, p, 0.f, VS);  // (columns in HC are never read)
      static_for<8>([&](auto Lc) {
        constexpr int L = decltype(Lc)::value;
        if constexpr ((HC >> L) & 1) {
          constexpr float wl = (float)(576 / dval(L));
#pragma unroll
          for (int i = 0; i < 4; ++i)  // rows (i, 7 - i) as one register pair per block (inv8p's row pattern)
            static_for<2>([&](auto Bc) {
              constexpr int B = decltype(Bc)::value;
              const float2 v = f2fma(make_float2(bpf<B>(H[i][L] + BIAS2), bpf<B>(H[7 - i][L] + BIAS2)), f2(wl),
                                     f2(-KF * wl));
              UHS[B][L][i] = v.x;
              UHS[B][L][7 - i] = v.y;
            });
        }
      });
      inverse2d_p<RM, HC>(VS, UHS, p.tab.pm1, p.tab.pmr, sq_row_s);
    } else {
      inverse2d_s<RM, HC>(V, UH, p.tab.pm1, sq_row_s);
    }
  } else {
    auto sq_row = [&](auto Ic, auto row) {
      using cuda::std::get;
      static_for<8>([&](auto Nc) {
        constexpr int N = decltype(Nc)::value;
        acc[N] = sqacc(get<N>(row), acc[N]);
      });
    };
    inverse2d_hc<RM, HC>(V, UH, sq_row);
  }
  const float2 s01 = f2add(acc[0], acc[1]), s23 = f2add(acc[2], acc[3]);
  const float2 s45 = f2add(acc[4], acc[5]), s67 = f2add(acc[6], acc[7]);
  return f2add(f2add(s01, s23), f2add(s45, s67));
}

// Residual form of the quantiser error (compile-time r = 64, SSE only; C4's case).  By the same
// orthogonality, x - x^ = C^T (Z - Z^) C: the kernel inverts the per-coefficient quantisation
// residual instead of forming x^ and subtracting it from the re-read pixels.  With
// Z - Z^ = q (Y / (q sqrt dd) - k) = q rho and D's row weights w = (1/sqrt8, 1/sqrt6, 1/2, 1/sqrt6,
// ...) folded into the butterfly (w_0 factored out, the ratios sqrt2 and 2/sqrt3 as FFMA2 immediates:
// the same 22 operations per 1-D pass), x - x^ = (q / 8) X'' where X'' is the weighted inverse of
// rho.  The DC path carries no ratio, so a DC-only residual is exact (pin P18 holds bit for bit).
constexpr float QW_S2 = 1.41421356f;   // w_2 / w_0 = sqrt 2
constexpr float QW_RO = 1.15470054f;   // w_1 / w_0 = 2 / sqrt 3
__device__ __forceinline__ void inv8w(const float2 (&v)[8], float2 (&o)[8]) {
  const float2 pp = f2add(v[0], v[4]), qq = f2sub(v[0], v[4]);
  const float2 a0 = f2fma(v[2], f2(QW_S2), pp), a3 = f2fma(v[2], f2(-QW_S2), pp);
  const float2 a1 = f2fma(v[6], f2(-QW_S2), qq), a2 = f2fma(v[6], f2(QW_S2), qq);
  const float2 b0 = f2add(f2add(v[1], v[3]), v[5]), b1 = f2sub(f2sub(v[1], v[5]), v[7]);
  const float2 b2 = f2add(f2sub(v[1], v[3]), v[7]), b3 = f2sub(f2sub(v[5], v[3]), v[7]);
  o[0] = f2fma(b0, f2(QW_RO), a0);
  o[7] = f2fma(b0, f2(-QW_RO), a0);
  o[1] = f2fma(b1, f2(QW_RO), a1);
  o[6] = f2fma(b1, f2(-QW_RO), a1);
  o[2] = f2fma(b2, f2(QW_RO), a2);
  o[5] = f2fma(b2, f2(-QW_RO), a2);
  o[3] = f2fma(b3, f2(QW_RO), a3);
  o[4] = f2fma(b3, f2(-QW_RO), a3);
}

// LO adds the low part of the reciprocal (y * lo): the residual of an exactly lossless coefficient
// stays ~1e-13 for any q.  Without it rho carries |Y / (q sqrt dd)| * 2^-24 of rounding (<= 7.6e-6 for
// the DC at q = 16; SSE relative error ~2e-6 on C4 frames) and the DC at q = 16 (1 / 128, a power
// of two) stays exact, so P18's constant frames are still bit-exact; one FFMA2 (two register-read
// cycles) less per coefficient pair.  The host picks LO for q < 4, where |Y / (q sqrt dd)| (up to
// 16320 / (4 q)) makes that rounding visible at the SSE bar (adct_api.cu).
// the same weighted graph per block on scalars with one-instruction butterflies: (x + w y, x - w y)
// with the uniform pairs (1, -1), (sqrt 2, -sqrt 2), (2 / sqrt 3, -2 / sqrt 3) — the same single-rounded
// fused products as inv8w
__device__ __forceinline__ void inv8ws(const float (&v)[8], float (&o)[8], float2 pm, float2 ps, float2 pr) {
  const float2 pq = ffma2_bfly(v[0], v[4], pm);      // pp, qq
  const float2 a03 = ffma2_bfly(pq.x, v[2], ps);     // pp +- s2 v2
  const float2 a21 = ffma2_bfly(pq.y, v[6], ps);     // qq +- s2 v6: (a2, a1)
  const float2 s13 = ffma2_bfly(v[1], v[3], pm);     // v1 +- v3
  const float2 s57 = ffma2_bfly(v[5], v[7], pm);     // v5 +- v7
  const float b0 = s13.x + v[5], b1 = v[1] - s57.x, b2 = s13.y + v[7], b3 = s57.y - v[3];
  const float2 o07 = ffma2_bfly(a03.x, b0, pr);
  const float2 o16 = ffma2_bfly(a21.y, b1, pr);
  const float2 o25 = ffma2_bfly(a21.x, b2, pr);
  const float2 o34 = ffma2_bfly(a03.y, b3, pr);
  o[0] = o07.x; o[7] = o07.y; o[1] = o16.x; o[6] = o16.y;
  o[2] = o25.x; o[5] = o25.y; o[3] = o34.x; o[4] = o34.y;
}

template <bool LO, int SM = 0>
__device__ __forceinline__ float2 compress_quant_resid(const uint32_t (&Y)[8][8], const CompressParams& p) {
  float2 U[8][8];  // column pass outputs [row][col]
  static_for<8>([&](auto Lc) {
    constexpr int L = decltype(Lc)::value;
    float2 v[8], o[8];
    static_for<8>([&](auto Kc) {
      constexpr int K = decltype(Kc)::value, c = wclass(K, L);
      const float2 y = f2add(biased_pair(Y[K][L]), f2(-KF));                  // Y, exact
      const float2 t = f2fma(y, f2(p.tab.cc[c]), f2(12582912.0f));           // 1.5 2^23 + k (exact decision, R10)
      const float2 k = f2add(t, f2(-12582912.0f));
      // rho = Y / (q sqrt dd) - k with the reciprocal as hi + lo: y hi - k is exact-ish in the fma
      // (near cancellation), y lo restores the rest — a DC residual that is 0 in exact arithmetic
      // stays ~1e-13 instead of ~1e-7 (lossless blocks keep SSE ~ 0)
      if constexpr (LO)
        v[K] = f2fma(y, f2(p.tab.sql[c]), f2fma(y, f2(p.tab.sq[c]), make_float2(-k.x, -k.y)));
      else
        v[K] = f2fma(y, f2(p.tab.sq[c]), make_float2(-k.x, -k.y));
    });
    if constexpr (SM == 1 || SM == 2) {
      float va[8], vb[8], oa[8], ob[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        va[k] = v[k].x;
        vb[k] = v[k].y;
      }
      inv8ws(va, oa, p.tab.pm1, p.tab.ps2, p.tab.pro);
      inv8ws(vb, ob, p.tab.pm1, p.tab.ps2, p.tab.pro);
#pragma unroll
      for (int i = 0; i < 8; ++i) U[i][L] = make_float2(oa[i], ob[i]);
    } else {
      inv8w(v, o);
#pragma unroll
      for (int i = 0; i < 8; ++i) U[i][L] = o[i];
    }
  });
  float2 acc[8];
#pragma unroll
  for (int n = 0; n < 8; ++n) acc[n] = f2(0.f);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if constexpr (SM != 0) {
      float ua[8], ub[8], oa[8], ob[8];
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        ua[l] = U[i][l].x;
        ub[l] = U[i][l].y;
      }
      inv8ws(ua, oa, p.tab.pm1, p.tab.ps2, p.tab.pro);
      inv8ws(ub, ob, p.tab.pm1, p.tab.ps2, p.tab.pro);
#pragma unroll
      for (int n = 0; n < 4; ++n) {  // outputs n, 7 - n of one block leave one butterfly as a pair
        acc[n] = f2fma(make_float2(oa[n], oa[7 - n]), make_float2(oa[n], oa[7 - n]), acc[n]);
        acc[4 + n] = f2fma(make_float2(ob[n], ob[7 - n]), make_float2(ob[n], ob[7 - n]), acc[4 + n]);
      }
    } else {
      float2 o[8];
      inv8w(U[i], o);
#pragma unroll
      for (int n = 0; n < 8; ++n) acc[n] = f2fma(o[n], o[n], acc[n]);
    }
  }
  const float2 s01 = f2add(acc[0], acc[1]), s23 = f2add(acc[2], acc[3]);
  const float2 s45 = f2add(acc[4], acc[5]), s67 = f2add(acc[6], acc[7]);
  return f2add(f2add(s01, s23), f2add(s45, s67));
}

// ------------------------------------------------------------------------------------------
// Fused compress kernel: every warp owns a TMA ring of ST stages and runs forward + inverse +
// error on each tile (one warp tile = 16 rows x 256 columns = one block pair per lane).
// Ring depth and the minimum resident CTAs per SM (register cap) are tuned per r
// (tools/microbench/tune_compress.cu): small r is latency/occupancy-sensitive,
// large r needs the registers.
// ------------------------------------------------------------------------------------------
// measured on B200 (profiles/r01_tune_compress.txt): small r wants occupancy, large r registers
#ifndef ADCT_ST_ALL
#define ADCT_ST_ALL 0  // A/B: force one ring depth for every zonal compress kernel
#endif
#ifndef ADCT_R1_ST
#define ADCT_R1_ST 3  // r = 1: 3-stage ring at 4 CTAs/SM, +1.4 % interleaved (profiles/r02_variants_r1_ring.txt)
#endif
#ifndef ADCT_R3_ST
#define ADCT_R3_ST 3
#endif
#ifndef ADCT_R1_MINB
#define ADCT_R1_MINB 4
#endif
constexpr int compress_stages(int R) {
  return ADCT_ST_ALL ? ADCT_ST_ALL : R == 1 ? ADCT_R1_ST : (R == 2 || R == 3) ? ADCT_R3_ST : 2;  // r = 2, 3: HBM-side bound
}
// residual form from this r on: cheaper once the discarded set is the smaller one;
// measured with the scalar-butterfly residual (profiles/r02_variants_resid_from.txt): r = 23 residual
// 0.615 vs direct 0.546 of HBM, r = 22 equal, r <= 21 direct
#ifndef ADCT_RESID_FROM
#define ADCT_RESID_FROM 23
#endif
constexpr int compress_resid_r(int R) { return R >= ADCT_RESID_FROM && R < 64; }
// output rows per tile that take the f16 error route (ALU -> FMA pipe rebalancing, compress_inv)
// measured on B200 (profiles/r01_tune_fhfma.txt): the FHFMA error route wins for every direct r
// (r = 1 keeps two rows on the f32 route to balance its ALU-light body)
#ifndef ADCT_F16_R1
#define ADCT_F16_R1 6
#endif
constexpr int compress_f16_rows(int R) { return R == 1 ? ADCT_F16_R1 : 8; }
// inverse output rows in two register-light groups (inverse2d_grouped)
#ifndef ADCT_GROUPED
#define ADCT_GROUPED 0
#endif
#ifndef ADCT_NOGROUP
#define ADCT_NOGROUP 0
#endif
constexpr bool compress_grouped(int R) { return !ADCT_NOGROUP && (ADCT_GROUPED || (R >= 11 && R < ADCT_RESID_FROM)); }
// runtime-mask / quantiser / reconstruction kernels (all 64 coefficients live)
#ifndef ADCT_MINB_QRES
#define ADCT_MINB_QRES 2
#endif
#ifndef ADCT_MINB_RT
#define ADCT_MINB_RT 2  // measured: 5-17 % faster than 3 (no spills), profiles/r01_variants_session3.txt
#endif
// measured on B200 (profiles/r01_tune_minb.txt): small r wants occupancy, mid r registers
#ifndef ADCT_MINB_RESID
#define ADCT_MINB_RESID 4
#endif
#ifndef ADCT_MINB_R3
#define ADCT_MINB_R3 3  // r = 2, 3 (3-stage ring): 4 CTAs/SM spilled (LDL/STL); 3 CTAs: r = 3 0.91 -> 0.96 of HBM (profiles/r02_variants_r3_minb.txt)
#endif
#ifndef ADCT_SM4_LO
#define ADCT_SM4_LO 15  // the per-block run-time loop flavour (SM = 4) for the grouped r in [LO, HI]
#endif
#ifndef ADCT_SM4_HI
#define ADCT_SM4_HI 22  // measured (profiles/r02_variants_sm4.txt): r = 15-22 +1-3 %, r <= 14 slower
#endif
#ifndef ADCT_RSM4_LO
#define ADCT_RSM4_LO 99  // the per-block loop for the residual form (no injected columns) in [LO, HI]:
                          // measured 5-9 % slower at r = 29..50 (profiles/r02_variants_sm4.txt), off
#endif
#ifndef ADCT_RSM4_HI
#define ADCT_RSM4_HI 0
#endif
#ifndef ADCT_MINB_SM4
#define ADCT_MINB_SM4 4
#endif
#ifndef ADCT_MINB_GRP
#define ADCT_MINB_GRP 4  // grouped mid r (11 <= r < ADCT_RESID_FROM)
#endif
#ifndef ADCT_MINB_DS
#define ADCT_MINB_DS 3  // direct form 4 <= r <= 10: 3 CTAs/SM, no spills (r = 6 +1 %, profiles/r02_variants_minb3.txt)
#endif
constexpr int compress_minb(int R) {
  // r = 64 (lossless, all 64 coefficients through the direct form): 2 CTAs/SM, no spills (4 spilled 824 B)
  return compress_resid_r(R) ? ADCT_MINB_RESID
         : (R == 1 ? ADCT_R1_MINB : (R == 2 || R == 3) ? ADCT_MINB_R3 : R == 64 ? 2 : (R >= 4 && R <= 10) ? ADCT_MINB_DS
            : (compress_grouped(R) && R >= ADCT_SM4_LO && R <= ADCT_SM4_HI) ? ADCT_MINB_SM4
            : compress_grouped(R) ? ADCT_MINB_GRP : 4);
}

#ifndef ADCT_QUANT_RING_R
#define ADCT_QUANT_RING_R 1
#endif
#ifndef ADCT_ZONAL_RING_R
#define ADCT_ZONAL_RING_R 0
#endif
// run-time-stage ring (one body copy) for the other large-body kernels (A/B: tools/time_variants.py)
#ifndef ADCT_BIG_RING_R
#define ADCT_BIG_RING_R 1
#endif
#ifndef ADCT_HYB_LO
#define ADCT_HYB_LO 12
#endif
#ifndef ADCT_HYB_HI
#define ADCT_HYB_HI 14
#endif
// measured per r (profiles/r02_variants_inverse_flavour*.txt, r02_variants_hybrid_mid_r.txt,
// r02_variants_low_high_r.txt): scalar butterflies for the ungrouped direct form (r <= 10, except
// r = 2-4, 7, 8 where f32x2 is 1-4 % faster) and the residual form (r >= 23: +6-9 %), the hybrid
// (f32x2 columns, scalar rows) for the grouped r = 12..14 (+2-5 %), the per-block run-time loop
// (SM = 4: one block's plane live, scalar butterflies) for r = 15..22 (+1-3 %), f32x2 for r = 11 and
// the quantiser
constexpr int sinv_mode(int R, int MODE, int RECON) {
  return ADCT_SINV >= 0 ? ADCT_SINV
         : (MODE == MODE_ZONAL && RECON == REC_NONE && compress_resid_r(R) && hcol_mask(R) == 0 &&
            R >= ADCT_RSM4_LO && R <= ADCT_RSM4_HI)                                                ? 4
         : (MODE == MODE_ZONAL && RECON == REC_NONE && R < RT && !compress_grouped(R) &&
            !(R >= 2 && R <= 4) && R != 7 && R != 8)                                               ? 1
         : (MODE == MODE_ZONAL && RECON == REC_NONE && compress_grouped(R) && R >= ADCT_SM4_LO && R <= ADCT_SM4_HI)
             ? 4
         : (MODE == MODE_ZONAL && RECON == REC_NONE && compress_grouped(R) && R >= ADCT_HYB_LO && R <= ADCT_HYB_HI)
             ? 3
             : 0;
}
template <int R, int MODE, int RECON, int ST = compress_stages(R),
          int MINB = (MODE == MODE_ZONAL && RECON == REC_NONE && R < RT) ? compress_minb(R)
                     : ((MODE == MODE_QUANT && RECON == REC_NONE && R == 64) ? ADCT_MINB_QRES : ADCT_MINB_RT),
          bool RES = (MODE == MODE_ZONAL && RECON == REC_NONE && R < RT && compress_resid_r(R)),
          int F16 = (MODE == MODE_ZONAL && RECON == REC_NONE && R < RT) ? compress_f16_rows(R) : 0,
          bool GRP = (MODE == MODE_ZONAL && RECON == REC_NONE && R < RT) ? compress_grouped(R) : false,
          bool MIRB = ADCT_MIRB && RECON == REC_NONE && ((MODE == MODE_ZONAL && R < RT) || (MODE == MODE_QUANT && R == 64)),
          bool QLO = false, int SM = sinv_mode(R, MODE, RECON)>
__global__ void __launch_bounds__(WARPS * 32, MINB)
    k_compress(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CompressParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  // errors in 576 units (ZONAL); the quantiser's residual form in units of q / 8 (compress_quant_resid)
  const double kSseScale = (MODE == MODE_ZONAL) ? 1.0 / 331776.0
                           : ((RECON == REC_NONE && R == 64) ? (double)p.tab.qscale : 1.0);
  // warp index through a shuffle: provably warp-uniform, so ptxas keeps the tile cursor in uniform
  // registers for the TMA (no per-lane R2UR loop)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (ST * TILE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * ST * TILE_BYTES) + warp * ST;
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  const float fxs = (float)(kSseScale * p.fx_scale);  // kernel units -> fixed-point pixel^2 units
  int cur = -1;
  long long acc = 0;
  auto tile_body = [&](const uint8_t* tile, int img, int ty, int tx) {
    if (img != cur) {  // warp-uniform: flush the finished image's partial SSE
      const long long v = warp_sum_ll(acc);
      if (lane == 0 && cur >= 0) fx_flush(p.sse + cur, v);
      cur = img;
      acc = 0;
    }
    uint32_t Y[8][8];
    float2 e2;
    if constexpr (RES) {
      constexpr int INJ = hcol_mask(R) | (ADCT_RESID_PC ? pcol_mask(R) : 0) | resid_p2_mask(R);
      if constexpr (ADCT_RESID_HC && INJ != 0 && !GRP) {
        uint32_t H[8][8];
        compress_fwd_h<RESID + R, INJ, MIRB>(tile, lane, Y, H);
        e2 = compress_resid_hc<R, SM>(Y, H, p);
      } else {
        compress_fwd<RESID + R, MODE, MIRB>(tile, lane, Y);
        e2 = compress_resid<R, GRP, SM>(Y, p);
      }
    } else if constexpr (MODE == MODE_QUANT && RECON == REC_NONE && R == 64) {
      compress_fwd<64, MODE, MIRB>(tile, lane, Y);
      e2 = compress_quant_resid<QLO, SM>(Y, p);
    } else {
      compress_fwd<R, MODE, MIRB>(tile, lane, Y);
      e2 = compress_inv<R, MODE, RECON, F16, GRP, false, MIRB, SM>(Y, tile, lane, p, img, ty, tx);
    }
    acc += fx_lane(e2, fxs);
  };
  // C4's quantiser body is ~1300 instructions: one copy of it (run-time ring stage) so the warps
  // do not stall on instruction fetch; the smaller zonal bodies keep the stage-unrolled ring
  if constexpr ((MODE == MODE_QUANT && RECON == REC_NONE && R == 64 && ADCT_QUANT_RING_R) ||
                (MODE == MODE_ZONAL && RECON == REC_NONE && R < RT && ADCT_ZONAL_RING_R) ||
                (R == RT && ADCT_BIG_RING_R))
    tma_ring_loop_r<ST>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane, tile_body);
  else
    tma_ring_loop_u<ST>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane, tile_body);
  const long long v = warp_sum_ll(acc);
  if (lane == 0 && cur >= 0) fx_flush(p.sse + cur, v);
}

// ------------------------------------------------------------------------------------------
// Exact zonal SSE (adct_compress_sse576): the same forward and runtime-mask inverse
// as k_compress<RT, ZONAL>, but every per-pixel error e = 576 x - R (an exact integer, |e| < 2^19,
// tools/exactness_bounds.py) is squared and summed in 64-bit integers, so the per-image result
// sum (576 x - R)^2 is bit-exact (no fp32 accumulation).  |e| <= 329205, so
// e^2 < 1.09e11 and the per-image sum stays below 2^63 (int64-safe) for h w <= 2^26 (host check).
// A parity / validation kernel, not the headline: 64-bit multiply-adds instead of FFMA2.
// ------------------------------------------------------------------------------------------
#ifndef ADCT_EXACT_BITS
#define ADCT_EXACT_BITS 1
#endif
#ifndef ADCT_EXACT_SINV
#define ADCT_EXACT_SINV 1
#endif
__device__ __forceinline__ unsigned long long sq_exact(float e) {
  // e + 1.5 * 2^23 is exact for |e| < 2^22 and its bit pattern is 0x4B400000 + e
  const int ei = __float_as_int(e + 12582912.0f) - 0x4B400000;
  return (unsigned long long)((long long)ei * (long long)ei);
}
// R = RT: the runtime mask (per-position weights, any r); R < RT: a compile-time mask (C5's r set,
// exact_parts.cu), per-class weights and the inverse pruned to the kept coefficients
template <int R = RT>
__device__ __forceinline__ unsigned long long compress_inv_exact(const uint32_t (&Y)[8][8], const uint8_t* tile,
                                                                 int lane, const CompressParams& p) {
  float2 V[64];
  static_for<64>([&](auto KLc) {
    constexpr int kl = decltype(KLc)::value, k = kl / 8, l = kl % 8;
    if constexpr (R == RT) {
      V[kl] = f2fma(biased_pair(Y[k][l]), f2(p.tab.w[kl].x), f2(p.tab.c[kl].x));  // W . M . Y, exact
    } else if constexpr (kept(R, k, l)) {
      constexpr int c = wclass(k, l);
      V[kl] = f2fma(biased_pair(Y[k][l]), f2(p.tab.wc[c]), f2(p.tab.cc[c]));  // W . Y (kept), exact
    }
  });
  unsigned long long acc = 0ull;
#if ADCT_EXACT_BITS
  // The error as the BIT PATTERN of one float (round 2): with 589824 + 1.5 2^23 injected at the DC
  // weight, the f16-route FMA gives v = R - 576 x + 1.5 2^23 (every graph node stays an integer
  // below 2^24, tools/exactness_bounds.py max 919 029 + 13 172 736), a float in [2^23, 2^24) whose
  // bits are b = 0x4B400000 - e (e = 576 x - R; -v and sign bit for rows the graph stores negated).
  // Per pixel: one IMAD.WIDE.U32 sum of b^2 (mod 2^64) and one 32-bit sum of b; per tile
  // sum e^2 = sum b^2 - 2 K sum b + n K^2 (mod 2^64) with sum b = n K - sum e recovered exactly
  // from its low 32 bits (|sum e| <= 128 * 329205 < 2^31): the same exact integer as sq_exact.
  V[0] = f2add(V[0], f2(13172736.0f));  // 589824 (f16 route) + 12582912 (1.5 2^23), exact
  unsigned long long b2p = 0ull, b2n = 0ull;  // sum b^2 mod 2^64 of stored-positive / -negated rows
  uint32_t s1p = 0u, s1n = 0u;                // sum b mod 2^32
  int np = 0, nn = 0;                         // compile-time after unrolling
  auto err_row = [&](auto Ic, auto row) {
    constexpr int I = decltype(Ic)::value;
    using cuda::std::get;
    const uint2 wa = lds64_reload(tile + I * TILE_W + lane * 8);
    const uint2 wb = lds64_reload(tile + (I + 8) * TILE_W + lane * 8);
    static_for<8>([&](auto Nc) {
      constexpr int N = decltype(Nc)::value;
      constexpr uint32_t sel = ((N >> 1) & 1) ? 0x4342u : 0x4140u;
      const uint32_t ha = __byte_perm(N < 4 ? wa.x : wa.y, p.h16magic, sel);
      const uint32_t hb = __byte_perm(N < 4 ? wb.x : wb.y, p.h16magic, sel);
      const float2 v = err_fh<N>(ha, hb, get<N>(row));
      const uint32_t ba = __float_as_uint(v.x), bb = __float_as_uint(v.y);
      if constexpr (cuda::std::is_same<cuda::std::decay_t<decltype(get<N>(row))>, FV<true>>::value) {
        b2n += (unsigned long long)ba * ba;
        b2n += (unsigned long long)bb * bb;
        s1n += ba + bb;
        nn += 2;
      } else {
        b2p += (unsigned long long)ba * ba;
        b2p += (unsigned long long)bb * bb;
        s1p += ba + bb;
        np += 2;
      }
    });
  };
  if constexpr (ADCT_EXACT_SINV) {  // per-block one-instruction butterflies (§7)
    auto err_row_s = [&](auto Ic, const auto& ra, const auto& rb) { err_row(Ic, join_rows(ra, rb)); };
    float2 UH[8][8];  // unused
    inverse2d_s<R>(V, UH, p.tab.pm1, err_row_s);
  } else {
    inverse2d<R>(V, err_row);
  }
  auto fold = [](unsigned long long b2, uint32_t s1, int n, uint32_t K) {
    const long long se = (long long)(int32_t)((uint32_t)n * K - s1);  // sum e (sign immaterial)
    const unsigned long long sb = (unsigned long long)n * K - (unsigned long long)se;  // exact sum b
    return b2 - 2ull * K * sb + (unsigned long long)n * K * K;  // mod 2^64
  };
  if (np) acc += fold(b2p, s1p, np, 0x4B400000u);
  if (nn) acc += fold(b2n, s1n, nn, 0xCB400000u);
#else
  auto err_row = [&](auto Ic, auto row) {
    constexpr int I = decltype(Ic)::value;
    using cuda::std::get;
    const uint2 wa = lds64_reload(tile + I * TILE_W + lane * 8);
    const uint2 wb = lds64_reload(tile + (I + 8) * TILE_W + lane * 8);
    static_for<8>([&](auto Nc) {
      constexpr int N = decltype(Nc)::value;
      const float2 e = rsub(px576b<false>(N < 4 ? wa.x : wa.y, N < 4 ? wb.x : wb.y, N & 3), get<N>(row));
      acc += sq_exact(e.x) + sq_exact(e.y);
    });
  };
  inverse2d<RT>(V, err_row);
#endif
  return acc;
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int ST, int R = RT>
__global__ void __launch_bounds__(WARPS * 32, ADCT_MINB_RT)
    k_compress_exact(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CompressParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (ST * TILE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * ST * TILE_BYTES) + warp * ST;
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  int cur = -1;
  unsigned long long acc = 0ull;
  tma_ring_loop<(bool)ADCT_BIG_RING_R, ST>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane,
                      [&](const uint8_t* tile, int img, int ty, int tx) {
    if (img != cur) {  // warp-uniform: flush the finished image's partial sum
      const unsigned long long v = warp_sum_u64(acc);
      if (lane == 0 && cur >= 0) atomicAdd(p.sse576 + cur, v);
      cur = img;
      acc = 0ull;
    }
    uint32_t Y[8][8];
    compress_fwd<R, MODE_ZONAL>(tile, lane, Y);
    acc += compress_inv_exact<R>(Y, tile, lane, p);
  });
  const unsigned long long v = warp_sum_u64(acc);
  if (lane == 0 && cur >= 0) atomicAdd(p.sse576 + cur, v);
}
// sse[i] = sse576[i] / 576^2 (pixel^2 units)
template <int UNUSED = 0>
__global__ void k_sse576_to_f64(const unsigned long long* __restrict__ in, double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)in[i] / 331776.0;
}

// fixed-point (two's complement int64, units 2^-k) -> fp64, in place
template <int UNUSED = 0>
__global__ void k_fx_to_f64(double* __restrict__ buf, int64_t n, double inv_scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = (double)__double_as_longlong(buf[i]) * inv_scale;
}

// ------------------------------------------------------------------------------------------
// Forward only: Y (int16 / int32) or Z (fp32) image-shaped.
// ------------------------------------------------------------------------------------------
template <int OUT>
__device__ __forceinline__ void tile_forward(const uint8_t* tile, int lane, const ForwardParams& p, int img,
                                             int ty, int tx) {
  constexpr uint32_t K = (OUT == OUT_F32) ? BIAS2 : 0x8000u;
  uint32_t P[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
    pack_rows(lds64(tile + i * TILE_W + lane * 8), lds64(tile + (i + 8) * TILE_W + lane * 8), P[i]);
  uint32_t Y[8][8];
  fwd2d<K, 64>(P, Y);
  const int col = tx * TILE_W + lane * 8;
  if (col >= p.w) return;
  uint8_t* base = p.coef + (int64_t)img * p.coef_img_stride;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int row = ty * TILE_H + b * 8 + k;
      if (row >= p.h) continue;
      uint8_t* rp = base + (int64_t)row * p.coef_pitch;
      if constexpr (OUT == OUT_I16) {
        uint32_t o[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          o[m] = b ? __byte_perm(Y[k][2 * m], Y[k][2 * m + 1], 0x7632)
                   : (__byte_perm(Y[k][2 * m], Y[k][2 * m + 1], 0x5410) ^ 0x80008000u);
          if (p.masked) o[m] &= p.m16[k * 4 + m];
        }
        *reinterpret_cast<uint4*>(rp + (int64_t)col * 2) = make_uint4(o[0], o[1], o[2], o[3]);
      } else if constexpr (OUT == OUT_I32) {
        int v[8];
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          v[l] = b ? ((int32_t)Y[k][l] >> 16) : ((int)(Y[k][l] & 0xFFFFu) - 32768);
          if (p.masked && !((p.keep_raster >> (k * 8 + l)) & 1ull)) v[l] = 0;
        }
        int4* q = reinterpret_cast<int4*>(rp + (int64_t)col * 4);
        q[0] = make_int4(v[0], v[1], v[2], v[3]);
        q[1] = make_int4(v[4], v[5], v[6], v[7]);
      } else {
        float v[8];
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          const float2 y = f2add(biased_pair(Y[k][l]), f2(-KF));
          v[l] = (b ? y.y : y.x) * p.sc[k * 8 + l];
        }
        float4* q = reinterpret_cast<float4*>(rp + (int64_t)col * 4);
        q[0] = make_float4(v[0], v[1], v[2], v[3]);
        q[1] = make_float4(v[4], v[5], v[6], v[7]);
      }
    }
  }
}

#ifndef ADCT_FWD_ST
#define ADCT_FWD_ST 3
#endif
#ifndef ADCT_FWD_MINB
#define ADCT_FWD_MINB 3
#endif
constexpr int FWD_ST = ADCT_FWD_ST, FWD_MINB = ADCT_FWD_MINB;  // ring depth, CTAs per SM
template <int OUT>
__global__ void __launch_bounds__(WARPS * 32, FWD_MINB)
    k_forward(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ ForwardParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (FWD_ST * TILE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * FWD_ST * TILE_BYTES) + warp * FWD_ST;
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  tma_ring_loop_u<FWD_ST>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane, [&](const uint8_t* tile, int img, int ty, int tx) {
    tile_forward<OUT>(tile, lane, p, img, ty, tx);
  });
}

// ------------------------------------------------------------------------------------------
// Forward to an int16 plane with TMA bulk-tensor stores: each warp writes its 16 x 256 tile of
// coefficients (8 KiB) into a warp-private shared-memory staging buffer and one elected lane
// stores it with cp.async.bulk.tensor (edges clipped by the tensor map), instead of 16 STG.128
// per lane.  NSTG staging buffers per warp: the buffer is rewritten only after the bulk store
// that read it NSTG tiles ago has finished reading (cp.async.bulk.wait_group.read).
// ------------------------------------------------------------------------------------------
#ifndef ADCT_FWDT_ST
#define ADCT_FWDT_ST 2
#endif
#ifndef ADCT_FWDT_NSTG
#define ADCT_FWDT_NSTG 2
#endif
#ifndef ADCT_FWDT_MINB
#define ADCT_FWDT_MINB 2
#endif
constexpr int FWDT_ST = ADCT_FWDT_ST;
constexpr int FWDT_BAR_BYTES = 128;  // mbarriers, padded so the staging buffers stay 128-B aligned
// staging per warp tile: int16 8 KiB (double-buffered), int32 / f32 16 KiB (single: 2 CTAs per SM)
constexpr int fwdt_nstg(int OUT) { return OUT == OUT_I16 ? ADCT_FWDT_NSTG : 1; }
constexpr int fwdt_tile_out_bytes(int OUT) { return OUT == OUT_I16 ? 2 * TILE_BYTES : 4 * TILE_BYTES; }
constexpr int fwdt_smem_bytes(int OUT) {
  return WARPS * FWDT_ST * TILE_BYTES + FWDT_BAR_BYTES + WARPS * fwdt_nstg(OUT) * fwdt_tile_out_bytes(OUT);
}
__device__ __forceinline__ void bulk_store_3d(const CUtensorMap* map, uint32_t src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)), "r"(src), "r"(x), "r"(y), "r"(z)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int OUT>
__global__ void __launch_bounds__(WARPS * 32, ADCT_FWDT_MINB)
    k_forward_tma(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap omap,
                  const __grid_constant__ ForwardParams p) {
  constexpr int NSTG = fwdt_nstg(OUT), OB = fwdt_tile_out_bytes(OUT);
  constexpr uint32_t K = (OUT == OUT_F32) ? BIAS2 : 0x8000u;
  extern __shared__ __align__(128) uint8_t smem[];
  static_assert(WARPS * FWDT_ST * 8 <= FWDT_BAR_BYTES, "mbarrier area");
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (FWDT_ST * TILE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * FWDT_ST * TILE_BYTES) + warp * FWDT_ST;
  uint8_t* stg = smem + WARPS * FWDT_ST * TILE_BYTES + FWDT_BAR_BYTES + warp * (NSTG * OB);
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  int sidx = 0;
  tma_ring_loop_u<FWDT_ST>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane,
                           [&](const uint8_t* tile, int img, int ty, int tx) {
    uint8_t* buf = stg + sidx * OB;
    uint32_t P[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      pack_rows(lds64(tile + i * TILE_W + lane * 8), lds64(tile + (i + 8) * TILE_W + lane * 8), P[i]);
    uint32_t Y[8][8];
    fwd2d<K, 64>(P, Y);
    if (lane == 0) bulk_wait_read<NSTG - 1>();  // the store that last read `buf` is done reading
    __syncwarp();
#pragma unroll
    for (int b = 0; b < 2; ++b) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint8_t* row = buf + (b * 8 + k) * (OB / TILE_H);
        if constexpr (OUT == OUT_I16) {
          uint32_t o[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            o[m] = b ? __byte_perm(Y[k][2 * m], Y[k][2 * m + 1], 0x7632)
                     : (__byte_perm(Y[k][2 * m], Y[k][2 * m + 1], 0x5410) ^ 0x80008000u);
            if (p.masked) o[m] &= p.m16[k * 4 + m];
          }
          *reinterpret_cast<uint4*>(row + lane * 16) = make_uint4(o[0], o[1], o[2], o[3]);
        } else if constexpr (OUT == OUT_I32) {
          int v[8];
#pragma unroll
          for (int l = 0; l < 8; ++l) {
            v[l] = b ? ((int32_t)Y[k][l] >> 16) : ((int)(Y[k][l] & 0xFFFFu) - 32768);
            if (p.masked && !((p.keep_raster >> (k * 8 + l)) & 1ull)) v[l] = 0;
          }
          int4* q = reinterpret_cast<int4*>(row + lane * 32);
          q[0] = make_int4(v[0], v[1], v[2], v[3]);
          q[1] = make_int4(v[4], v[5], v[6], v[7]);
        } else {
          float v[8];
#pragma unroll
          for (int l = 0; l < 8; ++l) {
            const float2 y = f2add(biased_pair(Y[k][l]), f2(-KF));
            v[l] = (b ? y.y : y.x) * p.sc[k * 8 + l];
          }
          float4* q = reinterpret_cast<float4*>(row + lane * 32);
          q[0] = make_float4(v[0], v[1], v[2], v[3]);
          q[1] = make_float4(v[4], v[5], v[6], v[7]);
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> bulk copy
    __syncwarp();
    if (lane == 0) bulk_store_3d(&omap, smem_u32(buf), tx * TILE_W, ty * TILE_H, img);
    if constexpr (NSTG > 1) sidx = (sidx + 1 == NSTG) ? 0 : sidx + 1;
  });
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------------------------------
// Inverse only: coefficient plane -> reconstruction (direct vectorised loads; no staging).
// ------------------------------------------------------------------------------------------
template <int IN>
__device__ __forceinline__ void load_coef_row(const uint8_t* rp, bool ok, float (&v)[8]) {
  if (!ok) {
#pragma unroll
    for (int l = 0; l < 8; ++l) v[l] = 0.f;
    return;
  }
  if constexpr (IN == OUT_I16) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(rp));
    const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      v[2 * m] = (float)(int16_t)(w4[m] & 0xFFFFu);
      v[2 * m + 1] = (float)(int16_t)(w4[m] >> 16);
    }
  } else if constexpr (IN == OUT_I32) {
    const int4 a = __ldg(reinterpret_cast<const int4*>(rp)), b = __ldg(reinterpret_cast<const int4*>(rp) + 1);
    v[0] = (float)a.x; v[1] = (float)a.y; v[2] = (float)a.z; v[3] = (float)a.w;
    v[4] = (float)b.x; v[5] = (float)b.y; v[6] = (float)b.z; v[7] = (float)b.w;
  } else {
    const float4 a = __ldg(reinterpret_cast<const float4*>(rp)), b = __ldg(reinterpret_cast<const float4*>(rp) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}

template <int IN, int RECON>
__global__ void __launch_bounds__(WARPS * 32, 3) k_inverse(const __grid_constant__ InverseParams p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int ES = (IN == OUT_I16) ? 2 : 4;
  for (int64_t t = (int64_t)blockIdx.x * WARPS + warp; t < p.tiles; t += (int64_t)gridDim.x * WARPS) {
    int img, ty, tx;
    p.geo.decode(t, img, ty, tx);
    const int col = tx * TILE_W + lane * 8;
    const bool cok = col < p.w;
    const uint8_t* base = p.coef + (int64_t)img * p.coef_img_stride + (int64_t)col * ES;
    float2 V[64];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float a[8], b[8];
      const int ra = ty * TILE_H + k, rb = ra + 8;
      load_coef_row<IN>(base + (int64_t)ra * p.coef_pitch, cok && ra < p.h, a);
      load_coef_row<IN>(base + (int64_t)rb * p.coef_pitch, cok && rb < p.h, b);
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        const uint32_t km = p.tab.keep[k * 8 + l];  // masked f32 NaN / Inf must not reach the block
        V[k * 8 + l] = __fmul2_rn(make_float2(__uint_as_float(__float_as_uint(a[l]) & km),
                                              __uint_as_float(__float_as_uint(b[l]) & km)), p.tab.w[k * 8 + l]);
      }
    }
    uint8_t* dbase = p.dst + (int64_t)img * p.dst_img_stride;
    inverse2d<RT>(V, [&](auto Ic, auto row) {
      constexpr int I = decltype(Ic)::value;
      float2 xr[8];
      static_for<8>([&](auto Nc) {
        constexpr int N = decltype(Nc)::value;
        xr[N] = val(cuda::std::get<N>(row));
      });
      store_recon_row<RECON, true, (IN == OUT_F32 ? U8_SAFE576R : U8_SAFE576)>(dbase, p.dst_pitch, p.h, p.w, ty * TILE_H + I, col, xr);
    });
  }
}

// Inverse from an int16 coefficient plane staged by TMA (16 x 256 coefficients = 8 KiB per warp
// tile, the same ring as the compress kernels): a lane's two blocks are rows 0-7 / 8-15 of its
// 8-column slice.  Coefficients become biased float pairs (xor 0x80008000, PRMT pairing A/B, the
// 2^23 magic) weighted by the runtime mask table, then the f32x2 inverse and the store.
template <int RECON>
__global__ void __launch_bounds__(WARPS * 32, 3)
    k_inverse_i16(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ InverseParams p) {
  constexpr int TB = 2 * TILE_BYTES;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (2 * TB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * 2 * TB) + warp * 2;
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  tma_ring_loop_u<2, TB>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane,
                     [&](const uint8_t* tile, int img, int ty, int tx) {
    float2 V[64];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint4 a = *reinterpret_cast<const uint4*>(tile + (k * TILE_W + lane * 8) * 2);
      const uint4 b = *reinterpret_cast<const uint4*>(tile + ((k + 8) * TILE_W + lane * 8) * 2);
      const uint32_t wa[4] = {a.x ^ 0x80008000u, a.y ^ 0x80008000u, a.z ^ 0x80008000u, a.w ^ 0x80008000u};
      const uint32_t wb[4] = {b.x ^ 0x80008000u, b.y ^ 0x80008000u, b.z ^ 0x80008000u, b.w ^ 0x80008000u};
#pragma unroll
      for (int m = 0; m < 4; ++m) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kl = k * 8 + 2 * m + h;
          const uint32_t P = __byte_perm(wa[m], wb[m], h ? 0x7632 : 0x5410);  // (A + 2^15) | (B + 2^15) << 16
          V[kl] = f2fma(biased_pair(P), f2(p.tab.w[kl].x), f2(p.tab.c[kl].x));  // w Y (0 if masked)
        }
      }
    }
    const int col = tx * TILE_W + lane * 8;
    uint8_t* dbase = p.dst + (int64_t)img * p.dst_img_stride;
    inverse2d<RT>(V, [&](auto Ic, auto row) {
      constexpr int I = decltype(Ic)::value;
      float2 xr[8];
      static_for<8>([&](auto Nc) {
        constexpr int N = decltype(Nc)::value;
        xr[N] = val(cuda::std::get<N>(row));
      });
      store_recon_row<RECON, true, U8_SAFE576>(dbase, p.dst_pitch, p.h, p.w, ty * TILE_H + I, col, xr);
    });
  });
}

// ------------------------------------------------------------------------------------------
// k_inverse_tma<IN, RECON>: inverse from an int16 / int32 / f32 coefficient plane with TMA bulk-tensor
// stores of the reconstruction: the warp's
// 16 x 256 output tile (f32: 16 KiB, u8: 4 KiB) is staged in shared memory row by row and stored
// by one elected lane; the staging buffer is rewritten only after the previous store has read it.
// ------------------------------------------------------------------------------------------
#ifndef ADCT_INVT_MINB
#define ADCT_INVT_MINB 1
#endif
constexpr int invt_stage_bytes(int RECON) { return RECON == REC_F32 ? 4 * TILE_BYTES : TILE_BYTES; }
constexpr int invt_in_bytes(int IN) { return IN == OUT_I16 ? 2 * TILE_BYTES : 4 * TILE_BYTES; }
constexpr int invt_smem_bytes(int IN, int RECON) {
  return WARPS * 2 * invt_in_bytes(IN) + FWDT_BAR_BYTES + WARPS * invt_stage_bytes(RECON);
}
// int16 / int32 / f32 coefficient planes in (TMA ring of 8 / 16 / 16 KiB tiles), reconstruction out
// through shared-memory staging + one TMA bulk-tensor store per tile.  Coefficients enter the f32x2
// inverse weighted by the runtime mask table: int16 through the biased-pair magic, int32 through
// an exact I2FP conversion (any int32), f32 (Z) directly with masked positions zeroed by their bits.
template <int IN, int RECON>
__global__ void __launch_bounds__(WARPS * 32, ADCT_INVT_MINB)
    k_inverse_tma(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap omap,
                  const __grid_constant__ InverseParams p) {
  constexpr int TB = invt_in_bytes(IN);
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (2 * TB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * 2 * TB) + warp * 2;
  uint8_t* buf = smem + WARPS * 2 * TB + FWDT_BAR_BYTES + warp * invt_stage_bytes(RECON);
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  tma_ring_loop_u<2, TB>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane,
                         [&](const uint8_t* tile, int img, int ty, int tx) {
    float2 V[64];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if constexpr (IN == OUT_I16) {
        const uint4 a = *reinterpret_cast<const uint4*>(tile + (k * TILE_W + lane * 8) * 2);
        const uint4 b = *reinterpret_cast<const uint4*>(tile + ((k + 8) * TILE_W + lane * 8) * 2);
        const uint32_t wa[4] = {a.x ^ 0x80008000u, a.y ^ 0x80008000u, a.z ^ 0x80008000u, a.w ^ 0x80008000u};
        const uint32_t wb[4] = {b.x ^ 0x80008000u, b.y ^ 0x80008000u, b.z ^ 0x80008000u, b.w ^ 0x80008000u};
#pragma unroll
        for (int m = 0; m < 4; ++m) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int kl = k * 8 + 2 * m + h;
            const uint32_t P = __byte_perm(wa[m], wb[m], h ? 0x7632 : 0x5410);  // (A + 2^15) | (B + 2^15) << 16
            V[kl] = f2fma(biased_pair(P), f2(p.tab.w[kl].x), f2(p.tab.c[kl].x));  // w Y (0 if masked)
          }
        }
      } else {
        const uint4* ra = reinterpret_cast<const uint4*>(tile + (k * TILE_W + lane * 8) * 4);
        const uint4* rb = reinterpret_cast<const uint4*>(tile + ((k + 8) * TILE_W + lane * 8) * 4);
        const uint4 a0 = ra[0], a1 = ra[1], b0 = rb[0], b1 = rb[1];
        const uint32_t av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const uint32_t bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          const int kl = k * 8 + l;
          if constexpr (IN == OUT_I32)  // exact int -> f32 conversion (I2FP) for any int32, then w Y
            V[kl] = __fmul2_rn(make_float2((float)(int)av[l], (float)(int)bv[l]), p.tab.w[kl]);
          else  // a masked position is zeroed by its bits (a NaN / Inf there must not reach the block)
            V[kl] = __fmul2_rn(make_float2(__uint_as_float(av[l] & p.tab.keep[kl]), __uint_as_float(bv[l] & p.tab.keep[kl])),
                               p.tab.w[kl]);
        }
      }
    }
    if (lane == 0) bulk_wait_read<0>();  // the previous tile's store has finished reading `buf`
    __syncwarp();
    inverse2d<RT>(V, [&](auto Ic, auto row) {
      constexpr int I = decltype(Ic)::value;
      float2 xr[8];
      static_for<8>([&](auto Nc) {
        constexpr int N = decltype(Nc)::value;
        xr[N] = val(cuda::std::get<N>(row));
      });
      stage_recon_row<RECON, true, (IN == OUT_F32 ? U8_SAFE576R : U8_SAFE576)>(buf, I, lane, xr);
    });
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) bulk_store_3d(&omap, smem_u32(buf), tx * TILE_W, ty * TILE_H, img);
  });
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------------------------------
// Fused compress with a reconstruction output (runtime mask / quantiser, f32 or u8): the warp's
// reconstruction tile is staged in shared memory and leaves through one TMA bulk-tensor store.
// ------------------------------------------------------------------------------------------
constexpr int crec_smem_bytes(int RECON) {
  return WARPS * 2 * TILE_BYTES + FWDT_BAR_BYTES + WARPS * recon_stage_bytes(RECON);
}
#ifndef ADCT_RECON_SM
#define ADCT_RECON_SM 0  // inverse flavour of the compile-time-r reconstruction kernels (A/B knob)
#endif
// R = RT: the runtime mask (any r, and the quantiser); R < RT: a compile-time zonal mask (C5's r set,
// recon_parts.cu) — the forward and the inverse pruned to the kept coefficients
template <int MODE, int RECON, int R = RT>
__global__ void __launch_bounds__(WARPS * 32, ADCT_MINB_RT)
    k_compress_recon(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap omap,
                     const __grid_constant__ CompressParams p) {
  static_assert(R == RT || MODE == MODE_ZONAL, "compile-time masks: zonal only");
  constexpr int ST = 2;
  extern __shared__ __align__(128) uint8_t smem[];
  const double kSseScale = (MODE == MODE_ZONAL) ? 1.0 / 331776.0 : 1.0;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (ST * TILE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * ST * TILE_BYTES) + warp * ST;
  uint8_t* buf = smem + WARPS * ST * TILE_BYTES + FWDT_BAR_BYTES + warp * recon_stage_bytes(RECON);
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  const float fxs = (float)(kSseScale * p.fx_scale);
  int cur = -1;
  long long acc = 0;
  tma_ring_loop<(bool)ADCT_BIG_RING_R, ST>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane,
                      [&](const uint8_t* tile, int img, int ty, int tx) {
    if (img != cur) {  // warp-uniform: flush the finished image's partial SSE
      const long long v = warp_sum_ll(acc);
      if (lane == 0 && cur >= 0) fx_flush(p.sse + cur, v);
      cur = img;
      acc = 0;
    }
    uint32_t Y[8][8];
    compress_fwd<R, MODE>(tile, lane, Y);
    if (lane == 0) bulk_wait_read<0>();  // the previous tile's store has finished reading `buf`
    __syncwarp();
    const float2 e2 = compress_inv<R, MODE, RECON, 0, false, true, false, (R < RT ? ADCT_RECON_SM : 0)>(
        Y, tile, lane, p, img, ty, tx, buf);
    acc += fx_lane(e2, fxs);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) bulk_store_3d(&omap, smem_u32(buf), tx * TILE_W, ty * TILE_H, img);
  });
  const long long v = warp_sum_ll(acc);
  if (lane == 0 && cur >= 0) fx_flush(p.sse + cur, v);
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------------------------------
// Dense comparator path: any 8x8 transform T as dense fp32 products — the
// exact DCT (the paper's reference curve), the SDCT sign(C)/(2 sqrt2) (P:78,
// P:288-289), the coarse C0/2 or a caller matrix.  Per block: Z = T X T^T, keep the
// first r zig-zag coefficients, X^ = T^T Z T (the transpose is the inverse for orthogonal T and
// the "approximate inversion" otherwise), per-image SSE accumulated in fp64.
// Column-at-a-time formulation: for each frequency column l,  u = X T[l]^T,  z = T u (column l
// of Z, masked),  w = T^T z,  X^ += w T[l]  — one 8x8 accumulator live; T read as constant-bank
// operands; pixels re-read from the staged tile.
// ------------------------------------------------------------------------------------------
struct DenseParams {
  TileGeo geo;
  double fx_scale;  // fixed-point scale of the deterministic per-image SSE (fx_lane / fx_flush)
  int64_t tiles;
  int cshift;
  int h, w;
  double* sse;
  float* recon;  // optional f32 reconstruction plane
  int64_t recon_pitch, recon_img_stride;
  uint64_t keep_raster;  // bit k*8+l: coefficient (k, l) kept
  float T[64];           // row-major T[m][n]
};

__device__ __forceinline__ float px_byte(uint2 wv, int j) {
  return (float)((j < 4 ? (wv.x >> (8 * j)) : (wv.y >> (8 * (j - 4)))) & 0xFFu);
}

__device__ __forceinline__ double dense_block_sse(const uint8_t* tile, int lane, int b, const DenseParams& p,
                                                  int img, int ty, int tx) {
  float Xh[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int n = 0; n < 8; ++n) Xh[i][n] = 0.f;
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    float u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint2 wv = lds64(tile + (b * 8 + i) * TILE_W + lane * 8);
      float a = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) a = fmaf(px_byte(wv, j), p.T[l * 8 + j], a);
      u[i] = a;
    }
    float z[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) a = fmaf(p.T[k * 8 + i], u[i], a);
      z[k] = ((p.keep_raster >> (k * 8 + l)) & 1ull) ? a : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float wi = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) wi = fmaf(p.T[k * 8 + i], z[k], wi);
#pragma unroll
      for (int n = 0; n < 8; ++n) Xh[i][n] = fmaf(wi, p.T[l * 8 + n], Xh[i][n]);
    }
  }
  if (p.recon) {
    const int col = tx * TILE_W + lane * 8, row0 = ty * TILE_H + b * 8;
    if (col < p.w && row0 < p.h) {
      uint8_t* base = reinterpret_cast<uint8_t*>(p.recon) + (int64_t)img * p.recon_img_stride + (int64_t)col * 4;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4* q = reinterpret_cast<float4*>(base + (int64_t)(row0 + i) * p.recon_pitch);
        q[0] = make_float4(Xh[i][0], Xh[i][1], Xh[i][2], Xh[i][3]);
        q[1] = make_float4(Xh[i][4], Xh[i][5], Xh[i][6], Xh[i][7]);
      }
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint2 wv = lds64(tile + (b * 8 + i) * TILE_W + lane * 8);
    float row = 0.f;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const float e = px_byte(wv, n) - Xh[i][n];
      row = fmaf(e, e, row);
    }
    acc += (double)row;
  }
  return acc;
}

template <int UNUSED = 0>
__global__ void __launch_bounds__(WARPS * 32, 3)
    k_compress_dense(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ DenseParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (STAGES * TILE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * STAGES * TILE_BYTES) + warp * STAGES;
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  int cur = -1;
  long long acc = 0;
  tma_ring_loop<(bool)ADCT_BIG_RING_R, STAGES>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane, [&](const uint8_t* tile, int img, int ty, int tx) {
    if (img != cur) {
      const long long v = warp_sum_ll(acc);
      if (lane == 0 && cur >= 0) fx_flush(p.sse + cur, v);
      cur = img;
      acc = 0;
    }
    acc += fx_of(dense_block_sse(tile, lane, 0, p, img, ty, tx) + dense_block_sse(tile, lane, 1, p, img, ty, tx),
                 p.fx_scale);
  });
  const long long v = warp_sum_ll(acc);
  if (lane == 0 && cur >= 0) fx_flush(p.sse + cur, v);
}

// ------------------------------------------------------------------------------------------
// Parseval sweep: one read of the images gives the SSE of EVERY triangular r.
// C = D C0 is orthogonal, so the zonal reconstruction error of a block equals the energy
// of its discarded orthonormal coefficients: 576^2 SSE = 576 * sum_{zz >= r} W Y^2 with
// W = 576 / (d_i d_j).  The kernel accumulates, per image, the exact integer energy
// E_s = sum_blocks sum_{k+l=s} W_kl Y_kl^2 of each anti-diagonal s = 0..14 (u64); for a
// triangular r = (s+1)(s+2)/2 the SSE is sum_{s' > s} E_s' / 576 = (E_total - sum_{s' <= s} E_s') / 576.  No inverse is computed, so this
// is NOT the fwd+zonal+inv path of the headline metric and is reported separately.
// ------------------------------------------------------------------------------------------
struct DiagParams {
  TileGeo geo;
  int64_t tiles;
  int cshift;
  int h, w;
  unsigned long long* energy;  // [n][16]
};

// weight groups of the anti-diagonals: position (k, l) -> index of W_kl among the distinct
// weights of anti-diagonal k + l (in order of first appearance), and the weight of group g
constexpr int diag_group_w(int s, int g) {
  int ws[4] = {0, 0, 0, 0}, n = 0;
  for (int k = 0; k < 8; ++k) {
    const int l = s - k;
    if (l < 0 || l > 7) continue;
    const int W = wval(k, l);
    bool seen = false;
    for (int i = 0; i < n; ++i) seen = seen || ws[i] == W;
    if (!seen) ws[n++] = W;
  }
  return g < n ? ws[g] : 0;
}
constexpr int diag_group(int k, int l) {
  for (int g = 0; g < 4; ++g)
    if (diag_group_w(k + l, g) == wval(k, l)) return g;
  return -1;
}

#ifndef ADCT_DIAG_ST
#define ADCT_DIAG_ST 2
#endif
#ifndef ADCT_DIAG_MINB
#define ADCT_DIAG_MINB 3
#endif
constexpr int DIAG_ST = ADCT_DIAG_ST, DIAG_MINB = ADCT_DIAG_MINB;  // ring depth, CTAs per SM (measured: 2/3 best, 0.53 vs 0.46 of HBM for 3/4)
// SMAX: the last anti-diagonal computed (14 = all; 7 = the triangular r <= 36 of C5, whose forward
// prunes the 28 coefficients of anti-diagonals 8..14).  Slot 15 of every image receives the block
// energy sum_all W Y^2 = 576 sum x^2 (P9 at r = 64: R = 576 x), from the pixels with one IDP4A per
// four (exact u32 per tile: 128 x 255^2 < 2^24), so SSE(r_s) = (E_15 - sum_{s' <= s} E_s') / 576
// needs only the anti-diagonals up to s.
template <int SMAX = 14>
__global__ void __launch_bounds__(WARPS * 32, DIAG_MINB)
    k_diag_energy(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ DiagParams p) {
  static_assert(SMAX >= 0 && SMAX <= 14, "anti-diagonals 0..14");
  constexpr int NS = SMAX + 1, RC = SMAX <= 7 ? (SMAX + 1) * (SMAX + 2) / 2 : 64;  // RC: zig-zag prefix
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (DIAG_ST * TILE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * DIAG_ST * TILE_BYTES) + warp * DIAG_ST;
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  int cur = -1;
  long long E[NS + 1];  // E[NS]: 576 sum x^2 (slot 15)
#pragma unroll
  for (int s = 0; s <= NS; ++s) E[s] = 0;
  auto flush = [&](int img) {
#pragma unroll
    for (int s = 0; s <= NS; ++s) {
      long long v = E[s];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && img >= 0) atomicAdd(p.energy + (int64_t)img * 16 + (s == NS ? 15 : s), (unsigned long long)v);
      E[s] = 0;
    }
  };
  tma_ring_loop<(bool)ADCT_BIG_RING_R, DIAG_ST>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane, [&](const uint8_t* tile, int img, int ty, int tx) {
    if (img != cur) {
      flush(cur);
      cur = img;
    }
    uint32_t P[8][8];
    uint32_t x2 = 0u;  // sum of the 128 squared pixels of this lane's block pair (IDP4A)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint2 wa = lds64(tile + i * TILE_W + lane * 8), wb = lds64(tile + (i + 8) * TILE_W + lane * 8);
      x2 = __dp4a(wa.x, wa.x, x2);
      x2 = __dp4a(wa.y, wa.y, x2);
      x2 = __dp4a(wb.x, wb.x, x2);
      x2 = __dp4a(wb.y, wb.y, x2);
      pack_rows(wa, wb, P[i]);
    }
    E[NS] += 576ll * (long long)x2;
    uint32_t Y[8][8];
    fwd2d<0u, RC>(P, Y);  // unbiased: lo lane = Y_A (two's complement), P - Y_A = Y_B * 2^16 exactly
    // Per tile, exact u32 sums of Y^2 per (anti-diagonal s, weight W) group — 28 groups, at most 4
    // positions x 2 blocks each, so a sum stays below 8 * 16320^2 < 2^32 — then one 64-bit
    // multiply-add E_s += W * S per group.  Per coefficient pair: Y_A = sext16 (PRMT), Y_A^2 (IMAD),
    // d = P - Y_A = Y_B 2^16 (IADD), Y_B^2 = hi(d * d) (IMAD.HI): 2 ALU + 2 FMA-pipe instructions.
    uint32_t S[NS][4];
    static_for<NS>([&](auto Sc) {
      static_for<4>([&](auto Gc) { S[decltype(Sc)::value][decltype(Gc)::value] = 0u; });
    });
    static_for<64>([&](auto KLc) {
      constexpr int kl = decltype(KLc)::value, k = kl / 8, l = kl % 8;
      if constexpr (k + l <= SMAX) {
        constexpr int g = diag_group(k, l);
        const uint32_t w = Y[k][l];
        const int a = (int)(int16_t)(w & 0xFFFFu);      // sign-extended low lane: Y of block A
        const int d = (int)(w - (uint32_t)a);           // Y of block B times 2^16
        S[k + l][g] += (uint32_t)(a * a) + (uint32_t)__mulhi(d, d);
      }
    });
    static_for<NS>([&](auto Sc) {
      constexpr int sd = decltype(Sc)::value;
      static_for<4>([&](auto Gc) {
        constexpr int g = decltype(Gc)::value;
        if constexpr (diag_group_w(sd, g) > 0)
          E[sd] += (long long)((unsigned long long)S[sd][g] * (unsigned)diag_group_w(sd, g));
      });
    });
  });
  flush(cur);
}

// SSE / PSNR of triangular r from the anti-diagonal energies: SSE(r_s) = sum_{s' > s} E_s' / 576.
struct SweepList {
  int n_r;
  int diag[16];  // anti-diagonal index s of each requested triangular r
};
template <int UNUSED = 0>
__global__ void k_sweep_psnr(const unsigned long long* __restrict__ energy, int64_t n, const __grid_constant__ SweepList L,
                             double pixels, double* __restrict__ sse, double* __restrict__ psnr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * L.n_r) return;
  const int64_t img = i % n;
  const int k = (int)(i / n);
  // SSE(r_s) = (E_15 - sum_{s' <= s} E_s') / 576 with E_15 = sum_all W Y^2 = 576 sum x^2 (exact in
  // u64); an anti-diagonal the energy kernel did not compute (UINT64_MAX) makes the result NaN
  unsigned long long acc = energy[img * 16 + 15];
  bool missing = false;
  for (int s = 0; s <= L.diag[k]; ++s) {
    const unsigned long long v = energy[img * 16 + s];
    missing = missing || v == ~0ull;
    acc -= v;
  }
  const double e = (double)acc / 576.0;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  sse[i] = missing ? nan : e;
  psnr[i] = missing ? nan : (acc == 0) ? __longlong_as_double(0x7ff0000000000000ll) : 10.0 * log10(65025.0 * pixels / e);
}

// ------------------------------------------------------------------------------------------
// Universal quality index: mean over all 8x8 sliding windows
// (stride 1) of Q = 4 C Mx My / ((Vx + Vy)(Mx^2 + My^2)) with C = N Sxy - Sx Sy,
// V = N S.. - S.^2, M = S. (window sums, N = 64; the normalisations cancel) = L * S with
// L = 2 Mx My / (Mx^2 + My^2), S = 2 C / (Vx + Vy); reading R16: a 0/0 factor is 1.
// x sums are exact integers, y sums fp64.  One CTA (256 threads) per 32x32 block of window
// origins: the 39x39 x / y patch is staged in shared memory, horizontal 8-sums per row, then
// vertical 8-sums per window.
// ------------------------------------------------------------------------------------------
constexpr int UQI_T = 32, UQI_P = UQI_T + 7;
struct UqiParams {
  const uint8_t* x;
  int64_t x_pitch, x_img_stride;
  const float* y;
  int64_t y_pitch, y_img_stride;
  int h, w, tiles_x, tiles_y;
  double inv_windows;  // 1 / ((h - 7)(w - 7))
  double fx_scale;     // fixed-point scale of the deterministic per-image mean (fx_lane / fx_flush)
  double* out;         // [n]
};

template <int UNUSED = 0>
__global__ void __launch_bounds__(256) k_uqi(const __grid_constant__ UqiParams p) {
  __shared__ int hx[UQI_P][UQI_T], hxx[UQI_P][UQI_T];
  __shared__ double hy[UQI_P][UQI_T], hyy[UQI_P][UQI_T], hxy[UQI_P][UQI_T];
  __shared__ uint8_t px[UQI_P][UQI_P + 1];
  __shared__ float py[UQI_P][UQI_P + 1];
  __shared__ double red[8];
  const int img = blockIdx.z, ty = blockIdx.y, tx = blockIdx.x;
  const int r0 = ty * UQI_T, c0 = tx * UQI_T;
  const uint8_t* xb = p.x + (int64_t)img * p.x_img_stride;
  const uint8_t* yb = reinterpret_cast<const uint8_t*>(p.y) + (int64_t)img * p.y_img_stride;
  for (int i = threadIdx.x; i < UQI_P * UQI_P; i += blockDim.x) {
    const int r = i / UQI_P, c = i % UQI_P, gr = r0 + r, gc = c0 + c;
    const bool ok = gr < p.h && gc < p.w;
    px[r][c] = ok ? xb[(int64_t)gr * p.x_pitch + gc] : 0;
    py[r][c] = ok ? *reinterpret_cast<const float*>(yb + (int64_t)gr * p.y_pitch + (int64_t)gc * 4) : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < UQI_P * UQI_T; i += blockDim.x) {
    const int r = i / UQI_T, c = i % UQI_T;
    int sx = 0, sxx = 0;
    double sy = 0, syy = 0, sxy = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int a = px[r][c + k];
      const double b = (double)py[r][c + k];
      sx += a;
      sxx += a * a;
      sy += b;
      syy = fma(b, b, syy);
      sxy = fma((double)a, b, sxy);
    }
    hx[r][c] = sx;
    hxx[r][c] = sxx;
    hy[r][c] = sy;
    hyy[r][c] = syy;
    hxy[r][c] = sxy;
  }
  __syncthreads();
  double q_acc = 0.0;
  for (int i = threadIdx.x; i < UQI_T * UQI_T; i += blockDim.x) {
    const int r = i / UQI_T, c = i % UQI_T;
    if (r0 + r > p.h - 8 || c0 + c > p.w - 8) continue;  // window must fit in the image
    long long Sx = 0, Sxx = 0;
    double Sy = 0, Syy = 0, Sxy = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      Sx += hx[r + k][c];
      Sxx += hxx[r + k][c];
      Sy += hy[r + k][c];
      Syy += hyy[r + k][c];
      Sxy += hxy[r + k][c];
    }
    const double Mx = (double)Sx, My = Sy;
    const double Vx = (double)(64 * Sxx - Sx * Sx);                // exact integer
    const double Vy = fmax(fma(64.0, Syy, -Sy * Sy), 0.0);
    const double C = fma(64.0, Sxy, -Mx * My);
    const double d1 = Vx + Vy, d2 = fma(Mx, Mx, My * My);
    // Q = L * S, a 0/0 factor taken as 1 (reading R16); guards 1e-12 pixel^2 = 4096e-12 in sum units
    const double L = (d2 <= 4.096e-9) ? 1.0 : 2.0 * Mx * My / d2;
    const double Sc = (d1 <= 4.096e-9) ? 1.0 : 2.0 * C / d1;
    const double q = L * Sc;
    q_acc += q;
  }
  q_acc = warp_sum(q_acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q_acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int k = 0; k < 8; ++k) t += red[k];
    fx_flush(p.out + img, fx_of(t * p.inv_windows, p.fx_scale));  // signed: two's complement wraps back
  }
}

// ------------------------------------------------------------------------------------------
// Fused multi-r sweep (with the inverse): one read and ONE forward per tile, then
// for every r of the set the full zonal step, inverse and per-pixel error (each r exactly the
// arithmetic of its own k_compress<r> instantiation: direct / grouped / residual form, f16 route).
// The forward is identical for every r, so computing it once is not work skipped; every r's
// reconstruction error is still computed pixel by pixel.  Reported separately from the headline
// (which runs the r-passes independently).  r are processed in descending order so the packed
// coefficients of the high anti-diagonals die early (register pressure).
// ------------------------------------------------------------------------------------------
struct RSetC5 {
  static constexpr int n = 8;
  static constexpr int r[8] = {36, 28, 21, 15, 10, 6, 3, 1};
};

#ifndef ADCT_MULTI_MINB
#define ADCT_MULTI_MINB 2
#endif
template <class RS>
__global__ void __launch_bounds__(WARPS * 32, ADCT_MULTI_MINB)
    k_compress_multi(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CompressParams p) {
  constexpr int ST = 2;
  constexpr double kSseScale = 1.0 / 331776.0;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (ST * TILE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * ST * TILE_BYTES) + warp * ST;
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  const float fxs = (float)(kSseScale * p.fx_scale);
  int cur = -1;
  long long acc[RS::n];
#pragma unroll
  for (int k = 0; k < RS::n; ++k) acc[k] = 0;
  auto flush = [&]() {
#pragma unroll
    for (int k = 0; k < RS::n; ++k) {
      const long long v = warp_sum_ll(acc[k]);
      if (lane == 0 && cur >= 0) fx_flush(p.sse + (int64_t)p.rowmap[k] * p.sse_stride + cur, v);
      acc[k] = 0;
    }
  };
  tma_ring_loop<(bool)ADCT_BIG_RING_R, ST>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane,
                      [&](const uint8_t* tile, int img, int ty, int tx) {
    if (img != cur) {  // warp-uniform
      flush();
      cur = img;
    }
    uint32_t Y[8][8];
    compress_fwd<64, MODE_ZONAL>(tile, lane, Y);  // all positions; outputs no r uses are dead code
    static_for<RS::n>([&](auto Kc) {
      constexpr int k = decltype(Kc)::value, R = RS::r[k];
      float2 e2;
      constexpr int SMR = sinv_mode(R, MODE_ZONAL, REC_NONE);
      if constexpr (compress_resid_r(R))
        e2 = compress_resid<R, compress_grouped(R), SMR>(Y, p);
      else
        e2 = compress_inv<R, MODE_ZONAL, REC_NONE, compress_f16_rows(R), compress_grouped(R), false, false, SMR>(
            Y, tile, lane, p, img, ty, tx);
      acc[k] += fx_lane(e2, fxs);
    });
  });
  flush();
}

// C0's entries at compile time, read off the same 22-addition graph as fwd8 applied to the unit
// vector e_i (so the sign patterns below can never disagree with the forward butterfly)
constexpr int c0_entry(int k, int i) {
  int x[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  x[i] = 1;
  const int a0 = x[0] + x[7], a1 = x[1] + x[6], a2 = x[2] + x[5], a3 = x[3] + x[4];
  const int b0 = x[0] - x[7], b1 = x[1] - x[6], b2 = x[2] - x[5], b3 = x[3] - x[4];
  const int X[8] = {a0 + a3 + a1 + a2, b0 + b1 + b2, a0 - a3, b0 - b2 - b3,
                    a0 + a3 - a1 - a2, b0 - b1 + b3, a2 - a1, b2 - b1 - b3};
  return X[k];
}

// Incremental fused sweep for C5's r set (the triangular numbers 1, 3, ..., 36: each adds one
// anti-diagonal b = 0..7 of the zig-zag mask).  R_r is linear in the kept coefficients, so with
// e = 576 x - R, e_{r_b} = e_{r_{b-1}} - dR_b where dR_b = C0^T (W . [band b] . Y) C0.  A band has
// one coefficient per column, so its column inverse is a sign pattern (T[k][i] V_kl, no adds) and
// only its row inverse costs butterfly adds; each r's error is still formed pixel by pixel
// (exactly, in integers < 2^24: tools/exactness_bounds.py, band variant) and squared.
template <int B, int I, int L> __device__ __forceinline__ auto band_in(const float2 (&V)[64]) {
  constexpr int k = B - L;
  if constexpr (k < 0 || k > 7) return Z0{};
  else if constexpr (c0_entry(k, I) == 0) return Z0{};
  else if constexpr (c0_entry(k, I) > 0) return FV<false>{V[k * 8 + L]};
  else return FV<true>{V[k * 8 + L]};
}
// the same for one block (scalar, one-instruction butterflies in the row inverse)
template <int B, int I, int L, int BLK> __device__ __forceinline__ auto band_in_s(const float2 (&V)[64]) {
  constexpr int k = B - L;
  if constexpr (k < 0 || k > 7) return Z0{};
  else if constexpr (c0_entry(k, I) == 0) return Z0{};
  else if constexpr (c0_entry(k, I) > 0) return SV<false>{BLK ? V[k * 8 + L].y : V[k * 8 + L].x};
  else return SV<true>{BLK ? V[k * 8 + L].y : V[k * 8 + L].x};
}
// the same from a per-block scalar plane (the split sweep)
template <int B, int I, int L> __device__ __forceinline__ auto band_in_v(const float (&VS)[64]) {
  constexpr int k = B - L;
  if constexpr (k < 0 || k > 7) return Z0{};
  else if constexpr (c0_entry(k, I) == 0) return Z0{};
  else if constexpr (c0_entry(k, I) > 0) return SV<false>{VS[k * 8 + L]};
  else return SV<true>{VS[k * 8 + L]};
}
__device__ __forceinline__ float ssub(float e, Z0) { return e; }
__device__ __forceinline__ float ssub(float e, SV<false> r) { return e - r.v; }
__device__ __forceinline__ float ssub(float e, SV<true> r) { return e + r.v; }
// e - (d_n, d_{7-n}) for ONE block: the pair (e_n, e_{7-n}) minus a band's row-inverse outputs n and
// 7 - n, which leave the same one-instruction butterfly as one register pair — one FADD2 / FFMA2 (two
// register reads) per two pixels instead of two scalar FADDs; a sign pair from a uniform register when
// the two outputs are stored with different signs (SV<neg>).  Exact: integers < 2^24 (R14).
__device__ __forceinline__ float2 esub2(float2 e, Z0, Z0, float2, float2) { return e; }
template <bool N> __device__ __forceinline__ float2 esub2(float2 e, SV<N> a, Z0, float2, float2) {
  return make_float2(ssub(e.x, a), e.y);
}
template <bool N> __device__ __forceinline__ float2 esub2(float2 e, Z0, SV<N> b, float2, float2) {
  return make_float2(e.x, ssub(e.y, b));
}
template <bool NA, bool NB>
__device__ __forceinline__ float2 esub2(float2 e, SV<NA> a, SV<NB> b, float2 pm, float2 pmr) {
  const float2 d = make_float2(a.v, b.v);
  if constexpr (NA == NB) return NA ? f2add(e, d) : f2sub(e, d);
  else if constexpr (NA) return __ffma2_rn(d, pm, e);  // (e.x + a, e.y - b)
  else return __ffma2_rn(d, pmr, e);                   // (e.x - a, e.y + b)
}
#ifndef ADCT_SWEEP_SINV
#define ADCT_SWEEP_SINV 1
#endif
#ifndef ADCT_SWEEP_PAIR
#define ADCT_SWEEP_PAIR 1  // per-block (n, 7 - n) error pairs (esub2) in the scalar-butterfly sweep
#endif

#ifndef ADCT_SWEEP_SPLIT
#define ADCT_SWEEP_SPLIT 1  // one block of the lane's pair at a time (fewer live registers)
#endif
#ifndef ADCT_SPLIT_UNROLL
#define ADCT_SPLIT_UNROLL 1
#endif
constexpr int kSplitUnroll = ADCT_SPLIT_UNROLL;
#ifndef ADCT_INC_MINB
#define ADCT_INC_MINB 2  // measured (profiles/r02_variants_sweep_split.txt): 2 > 3 > 4 CTAs/SM
#endif
template <int UNUSED = 0>
__global__ void __launch_bounds__(WARPS * 32, ADCT_INC_MINB)
    k_compress_sweep_inc(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CompressParams p) {
  constexpr int ST = 2, NB = 8;
  constexpr double kSseScale = 1.0 / 331776.0;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (ST * TILE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * ST * TILE_BYTES) + warp * ST;
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  const float fxs = (float)(kSseScale * p.fx_scale);
  int cur = -1;
  long long dacc[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) dacc[b] = 0;
  auto flush = [&]() {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const long long v = warp_sum_ll(dacc[b]);
      if (lane == 0 && cur >= 0) fx_flush(p.sse + (int64_t)p.rowmap[b] * p.sse_stride + cur, v);
      dacc[b] = 0;
    }
  };
  tma_ring_loop<(bool)ADCT_BIG_RING_R, ST>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane,
                      [&](const uint8_t* tile, int img, int ty, int tx) {
    if (img != cur) {  // warp-uniform
      flush();
      cur = img;
    }
    uint32_t Y[8][8];
    constexpr bool MIRB = ADCT_MIRB;  // block B column-mirrored (pack_rows_mirb): SSE only, errors mirrored
    compress_fwd<36, MODE_ZONAL, MIRB>(tile, lane, Y);
    if constexpr (ADCT_SWEEP_SPLIT) {
      // one block at a time: 36 scalar weighted coefficients live instead of 36 (A, B) pairs, so the
      // kernel fits 3 CTAs per SM without spills (the packed Y stays live for the second block)
      float2 acc[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) acc[b] = f2(0.f);
#pragma unroll (kSplitUnroll)
      for (int blk = 0; blk < 2; ++blk) {  // a run-time loop (unroll 1): ptxas keeps one block's plane live
        const uint32_t csel = blk ? 0x7632u : 0x7610u;
        float VS[64];
        static_for<64>([&](auto KLc) {
          constexpr int kl = decltype(KLc)::value, k = kl / 8, l = kl % 8;
          if constexpr (k + l < NB) {
            constexpr int c = wclass(k, l);
            VS[kl] = fmaf(__uint_as_float(__byte_perm(Y[k][l], 0x4B000000u, csel)), p.tab.wc[c], p.tab.cc[c]);
          }
        });
        const bool mir = MIRB && blk;  // block B column-mirrored: output column N is its pixel 7 - N
        static_for<8>([&](auto Ic) {
          constexpr int I = decltype(Ic)::value;
          const uint2 w = lds64_reload(tile + (I + 8 * blk) * TILE_W + lane * 8);
          auto px576 = [&](auto Nc) {  // 576 x for output column N
            constexpr int N = decltype(Nc)::value;
            constexpr uint32_t sel = ((N >> 1) & 1) ? 0x4342u : 0x4140u;
            constexpr uint32_t selm = ((N >> 1) & 1) ? 0x4041u : 0x4243u;
            const uint32_t word = ((N < 4) != mir) ? w.x : w.y;
            return fhfma576<(N & 1) != 0, true>(__byte_perm(word, p.h16magic, mir ? selm : sel), -DC_BIAS16);
          };
          float2 e[4];
          static_for<4>([&](auto Nc) {
            constexpr int N = decltype(Nc)::value;
            e[N] = make_float2(px576(cuda::std::integral_constant<int, N>{}),
                               px576(cuda::std::integral_constant<int, 7 - N>{}));
          });
          static_for<NB>([&](auto Bc) {
            constexpr int B = decltype(Bc)::value;
            auto rr = inv8s(band_in_v<B, I, 0>(VS), band_in_v<B, I, 1>(VS), band_in_v<B, I, 2>(VS),
                            band_in_v<B, I, 3>(VS), band_in_v<B, I, 4>(VS), band_in_v<B, I, 5>(VS),
                            band_in_v<B, I, 6>(VS), band_in_v<B, I, 7>(VS), p.tab.pm1);
            static_for<4>([&](auto Nc) {
              constexpr int N = decltype(Nc)::value;
              e[N] = esub2(e[N], cuda::std::get<N>(rr), cuda::std::get<7 - N>(rr), p.tab.pm1, p.tab.pmr);
              acc[B] = f2fma(e[N], e[N], acc[B]);
            });
          });
        });
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) dacc[b] += fx_lane(acc[b], fxs);
      return;
    }
    float2 V[64];
    static_for<64>([&](auto KLc) {
      constexpr int kl = decltype(KLc)::value, k = kl / 8, l = kl % 8;
      if constexpr (k + l < NB) {
        constexpr int c = wclass(k, l);
        V[kl] = f2fma(biased_pair(Y[k][l]), f2(p.tab.wc[c]), f2(p.tab.cc[c]));  // W . Y, exact
      }
    });
    float2 acc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[b] = f2(0.f);
    static_for<8>([&](auto Ic) {
      constexpr int I = decltype(Ic)::value;
      const uint2 wa = lds64_reload(tile + I * TILE_W + lane * 8);
      const uint2 wb = lds64_reload(tile + (I + 8) * TILE_W + lane * 8);
      if constexpr (ADCT_SWEEP_SINV && ADCT_SWEEP_PAIR) {
        // eA[n] = (e_n, e_{7-n}) of block A, eB likewise (B's pixels column-mirrored under MIRB)
        float2 eA[4], eB[4];
        auto px576 = [&](auto Nc, bool blkb) {
          constexpr int N = decltype(Nc)::value;
          constexpr uint32_t sel = ((N >> 1) & 1) ? 0x4342u : 0x4140u;
          constexpr uint32_t selb = MIRB ? (((N >> 1) & 1) ? 0x4041u : 0x4243u) : sel;
          if (!blkb) return fhfma576<(N & 1) != 0, true>(__byte_perm(N < 4 ? wa.x : wa.y, p.h16magic, sel), -DC_BIAS16);
          return fhfma576<(N & 1) != 0, true>(__byte_perm((N < 4) != MIRB ? wb.x : wb.y, p.h16magic, selb), -DC_BIAS16);
        };
        static_for<4>([&](auto Nc) {
          constexpr int N = decltype(Nc)::value;
          eA[N] = make_float2(px576(cuda::std::integral_constant<int, N>{}, false),
                              px576(cuda::std::integral_constant<int, 7 - N>{}, false));
          eB[N] = make_float2(px576(cuda::std::integral_constant<int, N>{}, true),
                              px576(cuda::std::integral_constant<int, 7 - N>{}, true));
        });
        static_for<NB>([&](auto Bc) {
          constexpr int B = decltype(Bc)::value;
          auto ra = inv8s(band_in_s<B, I, 0, 0>(V), band_in_s<B, I, 1, 0>(V), band_in_s<B, I, 2, 0>(V),
                          band_in_s<B, I, 3, 0>(V), band_in_s<B, I, 4, 0>(V), band_in_s<B, I, 5, 0>(V),
                          band_in_s<B, I, 6, 0>(V), band_in_s<B, I, 7, 0>(V), p.tab.pm1);
          auto rb = inv8s(band_in_s<B, I, 0, 1>(V), band_in_s<B, I, 1, 1>(V), band_in_s<B, I, 2, 1>(V),
                          band_in_s<B, I, 3, 1>(V), band_in_s<B, I, 4, 1>(V), band_in_s<B, I, 5, 1>(V),
                          band_in_s<B, I, 6, 1>(V), band_in_s<B, I, 7, 1>(V), p.tab.pm1);
          static_for<4>([&](auto Nc) {
            constexpr int N = decltype(Nc)::value;
            eA[N] = esub2(eA[N], cuda::std::get<N>(ra), cuda::std::get<7 - N>(ra), p.tab.pm1, p.tab.pmr);
            eB[N] = esub2(eB[N], cuda::std::get<N>(rb), cuda::std::get<7 - N>(rb), p.tab.pm1, p.tab.pmr);
            acc[B] = f2fma(eA[N], eA[N], acc[B]);
            acc[B] = f2fma(eB[N], eB[N], acc[B]);
          });
        });
      } else {  // (block A, block B) pairs: two scalar FADDs per pixel pair and band
        float2 e[8];  // 576 x - R of this output row, R over the bands added so far (none yet)
        static_for<8>([&](auto Nc) {
          constexpr int N = decltype(Nc)::value;
          // 576 (1024 + x) - 589824 = 576 x through the mixed-precision FMA (exact)
          constexpr uint32_t sel = ((N >> 1) & 1) ? 0x4342u : 0x4140u;
          constexpr uint32_t selb = MIRB ? (((N >> 1) & 1) ? 0x4041u : 0x4243u) : sel;
          const uint32_t ha = __byte_perm(N < 4 ? wa.x : wa.y, p.h16magic, sel);
          const uint32_t hb = __byte_perm((N < 4) != MIRB ? wb.x : wb.y, p.h16magic, selb);
          e[N] = make_float2(fhfma576<(N & 1) != 0, true>(ha, -DC_BIAS16), fhfma576<(N & 1) != 0, true>(hb, -DC_BIAS16));
        });
        static_for<NB>([&](auto Bc) {
          constexpr int B = decltype(Bc)::value;
          if constexpr (ADCT_SWEEP_SINV) {  // per block, one-instruction butterflies (inv8s)
            auto ra = inv8s(band_in_s<B, I, 0, 0>(V), band_in_s<B, I, 1, 0>(V), band_in_s<B, I, 2, 0>(V),
                            band_in_s<B, I, 3, 0>(V), band_in_s<B, I, 4, 0>(V), band_in_s<B, I, 5, 0>(V),
                            band_in_s<B, I, 6, 0>(V), band_in_s<B, I, 7, 0>(V), p.tab.pm1);
            auto rb = inv8s(band_in_s<B, I, 0, 1>(V), band_in_s<B, I, 1, 1>(V), band_in_s<B, I, 2, 1>(V),
                            band_in_s<B, I, 3, 1>(V), band_in_s<B, I, 4, 1>(V), band_in_s<B, I, 5, 1>(V),
                            band_in_s<B, I, 6, 1>(V), band_in_s<B, I, 7, 1>(V), p.tab.pm1);
            static_for<8>([&](auto Nc) {
              constexpr int N = decltype(Nc)::value;
              e[N] = make_float2(ssub(e[N].x, cuda::std::get<N>(ra)), ssub(e[N].y, cuda::std::get<N>(rb)));
              acc[B] = f2fma(e[N], e[N], acc[B]);
            });
          } else {
            auto row = inv8(band_in<B, I, 0>(V), band_in<B, I, 1>(V), band_in<B, I, 2>(V), band_in<B, I, 3>(V),
                            band_in<B, I, 4>(V), band_in<B, I, 5>(V), band_in<B, I, 6>(V), band_in<B, I, 7>(V));
            static_for<8>([&](auto Nc) {
              constexpr int N = decltype(Nc)::value;
              e[N] = rsub(e[N], cuda::std::get<N>(row));  // e_{r_B} = e_{r_{B-1}} - dR_B, exact
              acc[B] = f2fma(e[N], e[N], acc[B]);
            });
          }
        });
      }
    });
#pragma unroll
    for (int b = 0; b < NB; ++b) dacc[b] += fx_lane(acc[b], fxs);
  });
  flush();
}

// ------------------------------------------------------------------------------------------
// SDCT comparator on the integer fast path (F4 "reusing the integer machinery with
// a different T / D").  The SDCT is sign(C) / (2 sqrt 2) (reading R11) and its fast algorithm
// costs 24 additions per 1-D transform (Table 1).  With T_s = sign(C) (entries +-1):
//   Y = T_s X T_s^T (exact, |Y| <= 16320, the same packed 2 x int16 SWAR as the proposed forward),
//   Z = Y / 8, X^ = T^T (M_r . Z) T = R / 64 with R = T_s^T (M_r . Y) T_s (exact in fp32, |R| < 2^21),
//   e = 64 x - R per pixel (exact), SSE = sum e^2 / 4096.
// The SDCT is not orthogonal: X^ is the paper's "approximate inversion" by the transpose.
// Forward graph: a_n = x_n + x_{7-n}, b_n = x_n - x_{7-n}; even rows (+ + + +, + + - -, + - - +,
// + - + -) on a as a 4-point Hadamard; odd rows (+ + + +, + - - -, + - + +, + - + -) on b with
// t = b0 + b1, u = b0 - b1, v = b2 + b3, w = b2 - b3: X1 = t + v, X3 = u - v, X5 = u + v, X7 = u + w.
// ------------------------------------------------------------------------------------------
template <uint32_t K>
__device__ __forceinline__ void fwd8_sdct(const uint32_t (&x)[8], uint32_t (&X)[8]) {
  const uint32_t a0 = x[0] + x[7], a1 = x[1] + x[6], a2 = x[2] + x[5], a3 = x[3] + x[4];
  const uint32_t b0 = x[0] - x[7], b1 = x[1] - x[6], b2 = x[2] - x[5], b3 = x[3] - x[4];
  const uint32_t s01 = a0 + a1, d01 = a0 - a1, s23 = a2 + a3, d23 = a2 - a3;
  const uint32_t t = b0 + b1, u = b0 - b1, v = b2 + b3, w = b2 - b3;
  X[0] = s01 + s23 + K;
  X[2] = s01 - s23 + K;
  X[4] = d01 - d23 + K;
  X[6] = d01 + d23 + K;
  X[1] = t + v + K;
  X[3] = u - v + K;
  X[5] = u + v + K;
  X[7] = u + w + K;
}
// x = T_s^T X (transposed graph, 24 additions) on typed f32x2 values
template <class X0, class X1, class X2, class X3, class X4, class X5, class X6, class X7>
__device__ __forceinline__ auto inv8_sdct(X0 x0, X1 x1, X2 x2, X3 x3, X4 x4, X5 x5, X6 x6, X7 x7) {
  auto p = add(x0, x2), q = sub(x0, x2), r = add(x4, x6), s = sub(x4, x6);
  auto a0 = add(p, r), a1 = sub(p, r), a2 = sub(q, s), a3 = add(q, s);
  auto g = add(x1, x3), h = sub(x1, x3), i = add(x5, x7), j = sub(x5, x7);
  auto b0 = add(g, i), b1 = sub(h, i), b2 = add(h, i), b3 = add(h, j);
  return cuda::std::make_tuple(add(a0, b0), add(a1, b1), add(a2, b2), add(a3, b3), sub(a3, b3), sub(a2, b2),
                               sub(a1, b1), sub(a0, b0));
}
// the same graph per block with one-instruction butterflies: 11 butterflies + 2 scalar adds
template <class X0, class X1, class X2, class X3, class X4, class X5, class X6, class X7>
__device__ __forceinline__ auto inv8s_sdct(X0 x0, X1 x1, X2 x2, X3 x3, X4 x4, X5 x5, X6 x6, X7 x7, float2 pm) {
  using cuda::std::get;
  const auto pq = sbfly(x0, x2, pm);            // p = x0 + x2, q = x0 - x2
  const auto rs = sbfly(x4, x6, pm);            // r = x4 + x6, s = x4 - x6
  const auto a01 = sbfly(get<0>(pq), get<0>(rs), pm);  // a0 = p + r, a1 = p - r
  const auto a32 = sbfly(get<1>(pq), get<1>(rs), pm);  // a3 = q + s, a2 = q - s
  const auto gh = sbfly(x1, x3, pm);            // g = x1 + x3, h = x1 - x3
  const auto ij = sbfly(x5, x7, pm);            // i = x5 + x7, j = x5 - x7
  const auto b21 = sbfly(get<1>(gh), get<0>(ij), pm);  // b2 = h + i, b1 = h - i
  const auto b0 = add(get<0>(gh), get<0>(ij));
  const auto b3 = add(get<1>(gh), get<1>(ij));
  const auto o0 = sbfly(get<0>(a01), b0, pm);
  const auto o1 = sbfly(get<1>(a01), get<1>(b21), pm);
  const auto o2 = sbfly(get<1>(a32), get<0>(b21), pm);
  const auto o3 = sbfly(get<0>(a32), b3, pm);
  return cuda::std::make_tuple(get<0>(o0), get<0>(o1), get<0>(o2), get<0>(o3), get<1>(o3), get<1>(o2), get<1>(o1),
                               get<1>(o0));
}
#ifndef ADCT_SDCT_SINV
#define ADCT_SDCT_SINV 1
#endif

// e for pixel N of row (A, B) = R' -/+ 64 (1024 + x) through the mixed-precision FMA (exact):
// 0xD400 = f16(-64), 0x5400 = f16(+64)
template <bool HI, bool NEG>
__device__ __forceinline__ float fhfma64(uint32_t h2, float c) {
  float d;
  if constexpr (HI)
    asm("{.reg .f16 a, b; mov.b32 {_, a}, %1; mov.b16 b, %3; fma.rn.f32.f16 %0, a, b, %2;}"
        : "=f"(d) : "r"(h2), "f"(c), "n"(NEG ? 0x5400 : 0xD400));
  else
    asm("{.reg .f16 a, b; mov.b32 {a, _}, %1; mov.b16 b, %3; fma.rn.f32.f16 %0, a, b, %2;}"
        : "=f"(d) : "r"(h2), "f"(c), "n"(NEG ? 0x5400 : 0xD400));
  return d;
}
template <int N, bool NEG> __device__ __forceinline__ float2 err64(uint32_t ha, uint32_t hb, float2 v) {
  return make_float2(fhfma64<(N & 1) != 0, NEG>(ha, v.x), fhfma64<(N & 1) != 0, NEG>(hb, v.y));
}
constexpr float DC_BIAS64 = 65536.0f;  // 64 * 1024: injected at the DC (T_s row 0 is all ones)

template <int UNUSED = 0>
__global__ void __launch_bounds__(WARPS * 32, ADCT_MINB_RT)
    k_compress_sdct(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CompressParams p) {
  constexpr int ST = 2;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (ST * TILE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * ST * TILE_BYTES) + warp * ST;
  const StepPlan plan = make_step_plan(p.geo, p.tiles, p.cshift, (int)gridDim.x * WARPS);
  const float fxs = (float)(p.fx_scale / 4096.0);  // e = 64 (x - x^)
  int cur = -1;
  long long acc = 0;
  tma_ring_loop<(bool)ADCT_BIG_RING_R, ST>(&tmap, plan, (int)blockIdx.x * WARPS + warp, ring, bars, lane,
                      [&](const uint8_t* tile, int img, int ty, int tx) {
    if (img != cur) {
      const long long v = warp_sum_ll(acc);
      if (lane == 0 && cur >= 0) fx_flush(p.sse + cur, v);
      cur = img;
      acc = 0;
    }
    uint32_t P[8][8], H[8][8], Y[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      pack_rows(lds64(tile + i * TILE_W + lane * 8), lds64(tile + (i + 8) * TILE_W + lane * 8), P[i]);
#pragma unroll
    for (int i = 0; i < 8; ++i) fwd8_sdct<0u>(P[i], H[i]);
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      uint32_t c[8], o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = H[i][l];
      fwd8_sdct<BIAS2>(c, o);
#pragma unroll
      for (int k = 0; k < 8; ++k) Y[k][l] = o[k];
    }
    float2 V[64];  // M_r . Y (runtime mask as 0 / 1 weights), DC biased by 64 * 1024 for the f16 route
#pragma unroll
    for (int kl = 0; kl < 64; ++kl)
      V[kl] = f2fma(biased_pair(Y[kl / 8][kl % 8]), f2(p.tab.w[kl].x), f2(p.tab.c[kl].x + (kl == 0 ? DC_BIAS64 : 0.f)));
    float2 a2[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) a2[n] = f2(0.f);
    auto err_row = [&](auto Ic, const auto& row) {
      constexpr int I = decltype(Ic)::value;
      using cuda::std::get;
      const uint2 wa = lds64_reload(tile + I * TILE_W + lane * 8);
      const uint2 wb = lds64_reload(tile + (I + 8) * TILE_W + lane * 8);
      static_for<8>([&](auto Nc) {
        constexpr int N = decltype(Nc)::value;
        constexpr uint32_t sel = ((N >> 1) & 1) ? 0x4342u : 0x4140u;
        const uint32_t ha = __byte_perm(N < 4 ? wa.x : wa.y, p.h16magic, sel);
        const uint32_t hb = __byte_perm(N < 4 ? wb.x : wb.y, p.h16magic, sel);
        const auto rv = get<N>(row);
        const float2 e = err64<N, decltype(rv)::neg>(ha, hb, rv.v);  // R' - 64 (1024 + x) = R - 64 x, exact
        a2[N] = f2fma(e, e, a2[N]);
      });
    };
    auto col = [&](auto Lc) {
      constexpr int L = decltype(Lc)::value;
      return inv8_sdct(FV<false>{V[0 * 8 + L]}, FV<false>{V[1 * 8 + L]}, FV<false>{V[2 * 8 + L]}, FV<false>{V[3 * 8 + L]},
                       FV<false>{V[4 * 8 + L]}, FV<false>{V[5 * 8 + L]}, FV<false>{V[6 * 8 + L]}, FV<false>{V[7 * 8 + L]});
    };
    if constexpr (ADCT_SDCT_SINV) {
      auto cols = [&](auto Lc, auto Bc) {
        constexpr int L = decltype(Lc)::value, B = decltype(Bc)::value;
        auto g = [&](int k) { return SV<false>{B ? V[k * 8 + L].y : V[k * 8 + L].x}; };
        return inv8s_sdct(g(0), g(1), g(2), g(3), g(4), g(5), g(6), g(7), p.tab.pm1);
      };
      using I0 = cuda::std::integral_constant<int, 0>;
      using I1 = cuda::std::integral_constant<int, 1>;
      auto ua0 = cols(cuda::std::integral_constant<int, 0>{}, I0{}), ua1 = cols(cuda::std::integral_constant<int, 1>{}, I0{});
      auto ua2 = cols(cuda::std::integral_constant<int, 2>{}, I0{}), ua3 = cols(cuda::std::integral_constant<int, 3>{}, I0{});
      auto ua4 = cols(cuda::std::integral_constant<int, 4>{}, I0{}), ua5 = cols(cuda::std::integral_constant<int, 5>{}, I0{});
      auto ua6 = cols(cuda::std::integral_constant<int, 6>{}, I0{}), ua7 = cols(cuda::std::integral_constant<int, 7>{}, I0{});
      auto ub0 = cols(cuda::std::integral_constant<int, 0>{}, I1{}), ub1 = cols(cuda::std::integral_constant<int, 1>{}, I1{});
      auto ub2 = cols(cuda::std::integral_constant<int, 2>{}, I1{}), ub3 = cols(cuda::std::integral_constant<int, 3>{}, I1{});
      auto ub4 = cols(cuda::std::integral_constant<int, 4>{}, I1{}), ub5 = cols(cuda::std::integral_constant<int, 5>{}, I1{});
      auto ub6 = cols(cuda::std::integral_constant<int, 6>{}, I1{}), ub7 = cols(cuda::std::integral_constant<int, 7>{}, I1{});
      static_for<8>([&](auto Ic) {
        constexpr int I = decltype(Ic)::value;
        using cuda::std::get;
        auto ra = inv8s_sdct(get<I>(ua0), get<I>(ua1), get<I>(ua2), get<I>(ua3), get<I>(ua4), get<I>(ua5), get<I>(ua6),
                             get<I>(ua7), p.tab.pm1);
        auto rb = inv8s_sdct(get<I>(ub0), get<I>(ub1), get<I>(ub2), get<I>(ub3), get<I>(ub4), get<I>(ub5), get<I>(ub6),
                             get<I>(ub7), p.tab.pm1);
        err_row(Ic, join_rows(ra, rb));
      });
    } else {
    auto u0 = col(cuda::std::integral_constant<int, 0>{});
    auto u1 = col(cuda::std::integral_constant<int, 1>{});
    auto u2 = col(cuda::std::integral_constant<int, 2>{});
    auto u3 = col(cuda::std::integral_constant<int, 3>{});
    auto u4 = col(cuda::std::integral_constant<int, 4>{});
    auto u5 = col(cuda::std::integral_constant<int, 5>{});
    auto u6 = col(cuda::std::integral_constant<int, 6>{});
    auto u7 = col(cuda::std::integral_constant<int, 7>{});
    static_for<8>([&](auto Ic) {
      constexpr int I = decltype(Ic)::value;
      using cuda::std::get;
      auto row = inv8_sdct(get<I>(u0), get<I>(u1), get<I>(u2), get<I>(u3), get<I>(u4), get<I>(u5), get<I>(u6), get<I>(u7));
      err_row(Ic, row);
    });
    }
    const float2 s01 = f2add(a2[0], a2[1]), s23 = f2add(a2[2], a2[3]);
    const float2 s45 = f2add(a2[4], a2[5]), s67 = f2add(a2[6], a2[7]);
    acc += fx_lane(f2add(f2add(s01, s23), f2add(s45, s67)), fxs);
  });
  const long long v = warp_sum_ll(acc);
  if (lane == 0 && cur >= 0) fx_flush(p.sse + cur, v);
}

typedef void (*CompressKernel)(CUtensorMap, CompressParams);
// C4's quantiser kernel (compile-time r = 64, residual form) without / with the reciprocal's low part
template <bool LO> constexpr CompressKernel quant64_kernel() {
  return &k_compress<64, MODE_QUANT, REC_NONE, compress_stages(64), ADCT_MINB_QRES, false, 0, false,
                     (bool)ADCT_MIRB, LO, sinv_mode(64, MODE_QUANT, REC_NONE)>;
}
CompressKernel multi_kernel_c5();  // k_compress_multi<RSetC5>, instantiated in multi_r.cu
typedef void (*ReconKernel)(CUtensorMap, CUtensorMap, CompressParams);
CompressKernel exact_kernel(int r);  // compile-time-r exact-SSE kernels for C5's r set (exact_parts.cu)
ReconKernel zonal_recon_kernel(int r, int recon);  // compile-time-r reconstruction kernels (recon_parts.cu)
CompressKernel sweep_inc_kernel_c5();  // k_compress_sweep_inc, instantiated in multi_r.cu
// zonal kernels k_compress<r, ZONAL, RECON_NONE>, instantiated in zonal_part*.cu (4 TUs)
CompressKernel zonal_kernel(int r);

}  // namespace adct

