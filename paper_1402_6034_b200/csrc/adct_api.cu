// adct_api.cu — host side of the C ABI (include/adct.h): validation, TMA descriptors,
// per-call weight / quantiser tables, dispatch and launch.
#include "adct.h"

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>
#include "adct_kernels.cuh"

namespace adct {
__global__ void __launch_bounds__(256) k_psnr(const double* __restrict__ sse, int64_t count, double pixels,
                       double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double s = sse[i];
  out[i] = (s == 0.0) ? __longlong_as_double(0x7ff0000000000000ll)
                      : 10.0 * log10(65025.0 * pixels / s);
}
}  // namespace adct

// ==========================================================================================
// Host side: validation, tensor maps, dispatch, C ABI
// ==========================================================================================
namespace {

using namespace adct;

thread_local int g_last_cuda = 0;
thread_local int64_t g_launches = 0;

adct_status cuda_fail(cudaError_t e) {
  g_last_cuda = (int)e;
  return ADCT_ECUDA;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  // resolved once (thread-safe static initialisation), immutable afterwards
  static const EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(p);
    return static_cast<EncodeTiledFn>(nullptr);
  }();
  return fn;
}

adct_status make_u8_map(CUtensorMap* map, const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                        int64_t img_stride) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return cuda_fail(cudaErrorNotSupported);
  cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)img_stride};
  cuuint32_t box[3] = {TILE_W, TILE_H, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)src, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cuda_fail(cudaErrorInvalidValue);
  return ADCT_OK;
}

// int16 coefficient plane (adct_inverse's TMA path): same box, 2-byte elements (copied as UINT16 —
// TMA moves bytes; the kernel reinterprets them)
// image-shaped plane of 2- or 4-byte elements, one 16 x 256-element box per warp tile
adct_status make_plane_map(CUtensorMap* map, CUtensorMapDataType dt, const void* src, int64_t n, int64_t h,
                           int64_t w, int64_t pitch, int64_t img_stride) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return cuda_fail(cudaErrorNotSupported);
  cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)img_stride};
  cuuint32_t box[3] = {TILE_W, TILE_H, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, dt, 3, const_cast<void*>(src), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cuda_fail(cudaErrorInvalidValue);
  return ADCT_OK;
}
adct_status make_i16_map(CUtensorMap* map, const void* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                         int64_t img_stride) {
  return make_plane_map(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, src, n, h, w, pitch, img_stride);
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

adct_status check_geom(int64_t n, int64_t h, int64_t w) {
  if (n < 1 || h < 8 || w < 8 || (h & 7) || (w & 7)) return ADCT_EINVAL;
  if (n > INT32_MAX || h > INT32_MAX || w > INT32_MAX) return ADCT_EINVAL;
  // the device-side tile cursors are 32-bit: at most 2^30 tiles of 16 x 256 pixels per call
  const int64_t tiles = n * ((h + TILE_H - 1) / TILE_H) * ((w + TILE_W - 1) / TILE_W);
  if (tiles > (int64_t(1) << 30)) return ADCT_EINVAL;
  return ADCT_OK;
}

adct_status check_plane(const void* p, int64_t h, int64_t row_bytes, int64_t pitch, int64_t img_stride) {
  if (!p) return ADCT_EINVAL;
  if (pitch < row_bytes || img_stride < h * pitch) return ADCT_EINVAL;
  if (!aligned16(p) || (pitch & 15) || (img_stride & 15)) return ADCT_EALIGN;
  return ADCT_OK;
}

TileGeo make_geo(int64_t h, int64_t w) {
  TileGeo g;
  g.tiles_x = (w + TILE_W - 1) / TILE_W;
  g.tiles_y = (h + TILE_H - 1) / TILE_H;
  g.per_img = g.tiles_x * g.tiles_y;
  return g;
}

constexpr int zz_host(int i, int j) { return zz_index(i, j); }
double dd_host(int k, int l) { return (double)(dval(k) * dval(l)); }

// Smallest fp32 strictly above the exact 1 / (q sqrt(dd)): ties of the half-away rounding
// round away from zero (R10); compared exactly with 128-bit integers.
float quant_recip(float q, int dd) {
  auto above = [&](float c) {
    // c > 1/(q sqrt dd)  <=>  (c q)^2 dd > 1, with c = mc 2^ec, q = mq 2^eq exactly
    int ec, eq;
    double fc = frexp((double)c, &ec), fq = frexp((double)q, &eq);
    uint64_t mc = (uint64_t)ldexp(fc, 24), mq = (uint64_t)ldexp(fq, 24);
    ec -= 24;
    eq -= 24;
    unsigned __int128 m = (unsigned __int128)(mc * mq);  // < 2^48
    unsigned __int128 lhs = m * m * (unsigned __int128)dd;  // (c q)^2 dd = lhs * 2^(2(ec+eq))
    int e = 2 * (ec + eq);                                 // compare lhs * 2^e > 1
    if (e >= 0) return lhs > 0;
    int sh = -e;
    if (sh >= 127) return false;
    return lhs > ((unsigned __int128)1 << sh);
  };
  float c = (float)(1.0 / ((double)q * sqrt((double)dd)));
  while (above(nextafterf(c, 0.f))) c = nextafterf(c, 0.f);
  while (!above(c)) c = nextafterf(c, INFINITY);
  return c;
}

// the uniform multiplicand pairs of the one-instruction butterflies (adct_device.cuh inv8s / inv8ws)
void fill_bfly_pairs(Tables& t) {
  t.pm1 = make_float2(1.f, -1.f);
  t.pmr = make_float2(-1.f, 1.f);
  t.ps2 = make_float2(QW_S2, -QW_S2);
  t.pro = make_float2(QW_RO, -QW_RO);
}

void fill_zonal_tables(Tables& t, int r) {
  fill_bfly_pairs(t);
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l) {
      t.wc[wclass(k, l)] = (float)wval(k, l);
      t.cc[wclass(k, l)] = -KF * (float)wval(k, l);
    }
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l) {
      const bool keep = zz_host(k, l) < r;
      const float w = keep ? (float)wval(k, l) : 0.f;
      t.w[k * 8 + l] = make_float2(w, w);
      t.c[k * 8 + l] = make_float2(-KF * w, -KF * w);
    }
}

void fill_quant_tables(Tables& t, int r, float q) {
  fill_bfly_pairs(t);
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l) {
      const bool keep = zz_host(k, l) < r;
      // dequantised Z^ = q k enters the inverse as D Z^ D: q k / sqrt(d_k d_l) (x^ domain, fp32)
      const float qw = keep ? (float)((double)q / sqrt(dd_host(k, l))) : 0.f;
      const float c = quant_recip(q, dval(k) * dval(l));
      t.w[k * 8 + l] = make_float2(qw, qw);
      t.c[k * 8 + l] = make_float2(c, c);
      // per weight class (compile-time-r quantiser kernel): dequantiser weight and reciprocal
      t.wc[wclass(k, l)] = (float)((double)q / sqrt(dd_host(k, l)));
      t.cc[wclass(k, l)] = c;
      const double rq = 1.0 / ((double)q * sqrt(dd_host(k, l)));
      t.sq[wclass(k, l)] = (float)rq;
      t.sql[wclass(k, l)] = (float)(rq - (double)(float)rq);
    }
  t.qscale = (float)(((double)q / 8.0) * ((double)q / 8.0));
}

// Per (kernel, dynamic shared memory, device): the max-dynamic-smem attribute is set once and the
// resident-CTA count and SM count are remembered, so a call costs no occupancy query (host time
// per small call, profiles/r01_latency_c1.txt).  Thread-safe; entries are never removed.
struct LaunchShape {
  int sms, occ;
};
adct_status launch_shape(const void* kern, int smem, LaunchShape* out) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int>, LaunchShape> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  const auto key = std::make_tuple(kern, smem, dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return ADCT_OK;
    }
  }
  {
    // the attribute is a per-kernel maximum: raise it only, so a later launch of the same kernel
    // with a smaller shared-memory size cannot invalidate a cached larger one
    static std::map<std::pair<const void*, int>, int> attr_max;
    std::lock_guard<std::mutex> lock(mu);
    int& cur = attr_max[std::make_pair(kern, dev)];
    if (smem > cur) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return cuda_fail(e);
      cur = smem;
    }
  }
  LaunchShape ls{0, 0};
  cudaDeviceGetAttribute(&ls.sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ls.occ, kern, WARPS * 32, smem);
  if (e != cudaSuccess) return cuda_fail(e);
  if (ls.occ < 1) ls.occ = 1;
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = ls;
  *out = ls;
  return ADCT_OK;
}

template <class K, class P>
adct_status launch_tma_kernel(K kern, const CUtensorMap& map, const P& params_in, int64_t tiles,
                              cudaStream_t stream, int stages = STAGES, int tile_bytes = TILE_BYTES) {
  P params = params_in;
  const int smem = WARPS * stages * tile_bytes + WARPS * stages * 8;
  LaunchShape ls;
  adct_status st = launch_shape(reinterpret_cast<const void*>(kern), smem, &ls);
  if (st) return st;
  int64_t grid = (int64_t)ls.sms * ls.occ;
  // chunk = largest power of two <= 16 that still gives every resident warp >= 2 chunks
  int cshift = 4;
  while (cshift > 0 && (tiles >> cshift) < 2 * grid * WARPS) --cshift;
  params.cshift = cshift;
  const int64_t chunks = (tiles + (int64_t(1) << cshift) - 1) >> cshift;
  const int64_t need = (chunks + WARPS - 1) / WARPS;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, WARPS * 32, smem, stream>>>(map, params);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e);
}



// Kernels with an input and an output tensor map (TMA loads + TMA bulk stores).
template <class K, class P>
adct_status launch_tma2(K kern, const CUtensorMap& map, const CUtensorMap& omap, const P& params_in, int smem,
                        cudaStream_t stream) {
  P params = params_in;
  LaunchShape ls;
  adct_status st = launch_shape(reinterpret_cast<const void*>(kern), smem, &ls);
  if (st) return st;
  int64_t grid = (int64_t)ls.sms * ls.occ;
  int cshift = 4;
  while (cshift > 0 && (params.tiles >> cshift) < 2 * grid * WARPS) --cshift;
  params.cshift = cshift;
  const int64_t chunks = (params.tiles + (int64_t(1) << cshift) - 1) >> cshift;
  const int64_t need = (chunks + WARPS - 1) / WARPS;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, WARPS * 32, smem, stream>>>(map, omap, params);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e);
}
adct_status launch_forward_tma(adct_coef_t coef_t, const CUtensorMap& map, const CUtensorMap& omap,
                               const ForwardParams& p, cudaStream_t stream) {
  switch (coef_t) {
    case ADCT_COEF_I16: return launch_tma2(k_forward_tma<OUT_I16>, map, omap, p, fwdt_smem_bytes(OUT_I16), stream);
    case ADCT_COEF_I32: return launch_tma2(k_forward_tma<OUT_I32>, map, omap, p, fwdt_smem_bytes(OUT_I32), stream);
    default: return launch_tma2(k_forward_tma<OUT_F32>, map, omap, p, fwdt_smem_bytes(OUT_F32), stream);
  }
}

// Fixed-point exponent k of the deterministic per-image sums (fx_lane in adct_kernels.cuh): the largest
// possible per-image total, pixels * 2^bound_log2 (pixel^2 units), times 2^k stays below 2^61.
// Zonal / quantiser SSE: C = D C0 is orthogonal, so a block's error energy is at most the
// energy of its discarded / quantisation-residual coefficients, |Z - q k| <= |Z|, hence at most the
// block's own energy sum x^2 <= 64 * 255^2: bound_log2 = 17 leaves a factor 2 of headroom.
int fx_exponent(int64_t pixels, int bound_log2) {
  int lp = 0;
  while ((int64_t(1) << lp) < pixels) ++lp;
  int k = 61 - lp - bound_log2;
  return k < 0 ? 0 : (k > 60 ? 60 : k);
}
// in-place fixed-point -> fp64 conversion of n per-image sums after the accumulating kernel
adct_status fx_finish(double* buf, int64_t n, int k, cudaStream_t s) {
  const int64_t blocks = (n + 255) / 256;
  k_fx_to_f64<0><<<(unsigned)(blocks < 1024 ? blocks : 1024), 256, 0, s>>>(buf, n, ldexp(1.0, -k));
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e);
}
constexpr int FX_BOUND_SSE = 17;

// Compress launch: ring depth from the kernel's per-r configuration.
adct_status launch_compress(CompressKernel kern, int RF, const CUtensorMap& map, const CompressParams& p,
                            cudaStream_t stream) {
  return launch_tma_kernel(kern, map, p, p.tiles, stream, compress_stages(RF));
}

// the kernel choice of adct_compress_psnr (tables filled here; SSE buffer zeroed by the caller)
adct_status compress_dispatch(const CUtensorMap& map, const CUtensorMap& omap, bool bulk, CompressParams& p, int r,
                              float q, adct_recon_t recon_t, cudaStream_t s) {
  if (q > 0.f) {
    fill_quant_tables(p.tab, r, q);
    if (bulk && recon_t == ADCT_RECON_F32)
      return launch_tma2(k_compress_recon<MODE_QUANT, REC_F32>, map, omap, p, crec_smem_bytes(REC_F32), s);
    if (bulk) return launch_tma2(k_compress_recon<MODE_QUANT, REC_U8>, map, omap, p, crec_smem_bytes(REC_U8), s);
    if (recon_t == ADCT_RECON_NONE && r == 64)  // C4's case: compile-time mask, per-class constants
      return launch_compress(q < 4.f ? quant64_kernel<true>() : quant64_kernel<false>(), 64, map, p, s);
    if (recon_t == ADCT_RECON_NONE) return launch_compress(k_compress<RT, MODE_QUANT, REC_NONE>, RT, map, p, s);
    if (recon_t == ADCT_RECON_F32) return launch_compress(k_compress<RT, MODE_QUANT, REC_F32>, RT, map, p, s);
    return launch_compress(k_compress<RT, MODE_QUANT, REC_U8>, RT, map, p, s);
  }
  fill_zonal_tables(p.tab, r);
  if (recon_t == ADCT_RECON_NONE) {
    return launch_compress(zonal_kernel(r), r, map, p, s);
  }
  if (bulk) {  // C5's r: compile-time mask (pruned forward / inverse); any other r: the runtime mask
    const int rt = recon_t == ADCT_RECON_F32 ? REC_F32 : REC_U8;
    if (ReconKernel k = zonal_recon_kernel(r, rt)) return launch_tma2(k, map, omap, p, crec_smem_bytes(rt), s);
  }
  if (bulk && recon_t == ADCT_RECON_F32)
    return launch_tma2(k_compress_recon<MODE_ZONAL, REC_F32>, map, omap, p, crec_smem_bytes(REC_F32), s);
  if (bulk) return launch_tma2(k_compress_recon<MODE_ZONAL, REC_U8>, map, omap, p, crec_smem_bytes(REC_U8), s);
  if (recon_t == ADCT_RECON_F32) return launch_compress(k_compress<RT, MODE_ZONAL, REC_F32>, RT, map, p, s);
  return launch_compress(k_compress<RT, MODE_ZONAL, REC_U8>, RT, map, p, s);
}


}  // namespace

extern "C" {

const char* adct_status_string(adct_status s) {
  switch (s) {
    case ADCT_OK: return "ok";
    case ADCT_EINVAL: return "invalid argument";
    case ADCT_EALIGN: return "misaligned pointer, pitch or stride (16-byte rule)";
    case ADCT_ECUDA: return "CUDA error";
  }
  return "unknown status";
}

int adct_last_cuda_error(void) { return g_last_cuda; }
int adct_version(void) { return 10200; }
int64_t adct_launch_count(void) { return g_launches; }

adct_status adct_forward(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                         int64_t img_stride, int r, void* coef, adct_coef_t coef_t, int64_t coef_pitch,
                         int64_t coef_img_stride, adct_stream_t stream) {
  adct_status st = check_geom(n, h, w);
  if (st) return st;
  if (r < 1 || r > 64) return ADCT_EINVAL;
  if (coef_t != ADCT_COEF_I16 && coef_t != ADCT_COEF_I32 && coef_t != ADCT_COEF_F32) return ADCT_EINVAL;
  if ((st = check_plane(src, h, w, pitch, img_stride))) return st;
  const int es = coef_t == ADCT_COEF_I16 ? 2 : 4;
  if ((st = check_plane(coef, h, w * es, coef_pitch, coef_img_stride))) return st;
  CUtensorMap map;
  if ((st = make_u8_map(&map, src, n, h, w, pitch, img_stride))) return st;
  ForwardParams p;
  memset(&p, 0, sizeof(p));
  p.geo = make_geo(h, w);
  p.tiles = p.geo.per_img * n;
  p.h = (int)h;
  p.w = (int)w;
  p.coef = (uint8_t*)coef;
  p.coef_pitch = coef_pitch;
  p.coef_img_stride = coef_img_stride;
  p.masked = r < 64;
  p.keep_raster = 0;
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l)
      if (zz_host(k, l) < r) p.keep_raster |= 1ull << (k * 8 + l);
  for (int k = 0; k < 8; ++k)
    for (int m = 0; m < 4; ++m) {
      uint32_t mk = 0;
      if (zz_host(k, 2 * m) < r) mk |= 0xFFFFu;
      if (zz_host(k, 2 * m + 1) < r) mk |= 0xFFFF0000u;
      p.m16[k * 4 + m] = mk;
    }
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l)
      p.sc[k * 8 + l] = (zz_host(k, l) < r) ? (float)(1.0 / sqrt(dd_host(k, l))) : 0.f;
  cudaStream_t s = (cudaStream_t)stream;
#ifndef ADCT_FWD_TMA_STORE
#define ADCT_FWD_TMA_STORE 1
#endif
  if (ADCT_FWD_TMA_STORE) {  // coefficient tiles leave through shared memory + TMA bulk stores
    CUtensorMap omap;
    st = make_plane_map(&omap,
                        coef_t == ADCT_COEF_I16 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                        : coef_t == ADCT_COEF_I32 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        coef, n, h, w, coef_pitch, coef_img_stride);
    if (st) return st;
    return launch_forward_tma(coef_t, map, omap, p, s);
  }
  switch (coef_t) {
    case ADCT_COEF_I16: return launch_tma_kernel(k_forward<OUT_I16>, map, p, p.tiles, s, FWD_ST);
    case ADCT_COEF_I32: return launch_tma_kernel(k_forward<OUT_I32>, map, p, p.tiles, s, FWD_ST);
    default: return launch_tma_kernel(k_forward<OUT_F32>, map, p, p.tiles, s, FWD_ST);
  }
}

adct_status adct_inverse(const void* coef, adct_coef_t coef_t, int64_t n, int64_t h, int64_t w,
                         int64_t coef_pitch, int64_t coef_img_stride, int r, void* dst, adct_recon_t dst_t,
                         int64_t dst_pitch, int64_t dst_img_stride, adct_stream_t stream) {
  adct_status st = check_geom(n, h, w);
  if (st) return st;
  if (r < 1 || r > 64) return ADCT_EINVAL;
  if (coef_t != ADCT_COEF_I16 && coef_t != ADCT_COEF_I32 && coef_t != ADCT_COEF_F32) return ADCT_EINVAL;
  if (dst_t != ADCT_RECON_F32 && dst_t != ADCT_RECON_U8) return ADCT_EINVAL;
  const int es = coef_t == ADCT_COEF_I16 ? 2 : 4;
  if ((st = check_plane(coef, h, w * es, coef_pitch, coef_img_stride))) return st;
  if ((st = check_plane(dst, h, w * (dst_t == ADCT_RECON_F32 ? 4 : 1), dst_pitch, dst_img_stride))) return st;
  InverseParams p;
  memset(&p, 0, sizeof(p));
  p.geo = make_geo(h, w);
  p.tiles = p.geo.per_img * n;
  p.h = (int)h;
  p.w = (int)w;
  p.coef = (const uint8_t*)coef;
  p.coef_pitch = coef_pitch;
  p.coef_img_stride = coef_img_stride;
  p.dst = (uint8_t*)dst;
  p.dst_pitch = dst_pitch;
  p.dst_img_stride = dst_img_stride;
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l) {
      float m = 0.f;
      if (zz_host(k, l) < r)
        m = (coef_t == ADCT_COEF_F32) ? (float)(576.0 / sqrt(dd_host(k, l))) : (float)wval(k, l);
      p.tab.w[k * 8 + l] = make_float2(m, m);
      p.tab.c[k * 8 + l] = make_float2(-KF * m, -KF * m);  // TMA int16 path: debias of the magic pair
      p.tab.keep[k * 8 + l] = zz_host(k, l) < r ? 0xFFFFFFFFu : 0u;
    }
  cudaStream_t s0 = (cudaStream_t)stream;
#ifndef ADCT_INV_TMA_STORE
#define ADCT_INV_TMA_STORE 1
#endif
  // coefficient tiles in through the TMA rings, reconstruction tiles out through shared memory +
  // TMA bulk stores.  Measured on B200: a bulk tensor store writes a row's last partial 16-byte
  // chunk whole, so the u8 plane takes this path only when w is a multiple of 16
  // (tests/test_gpu_parity.py::test_no_writes_outside_outputs)
  if (ADCT_INV_TMA_STORE && (dst_t == ADCT_RECON_F32 || (w & 15) == 0)) {
    CUtensorMap map, omap;
    const CUtensorMapDataType it = coef_t == ADCT_COEF_I16 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                   : coef_t == ADCT_COEF_I32 ? CU_TENSOR_MAP_DATA_TYPE_INT32
                                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    if ((st = make_plane_map(&map, it, coef, n, h, w, coef_pitch, coef_img_stride))) return st;
    if (dst_t == ADCT_RECON_F32)
      st = make_plane_map(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, dst, n, h, w, dst_pitch, dst_img_stride);
    else
      st = make_u8_map(&omap, (const uint8_t*)dst, n, h, w, dst_pitch, dst_img_stride);
    if (st) return st;
#define ADCT_INVT(IN, RC) launch_tma2(k_inverse_tma<IN, RC>, map, omap, p, invt_smem_bytes(IN, RC), s0)
    if (coef_t == ADCT_COEF_I16) return dst_t == ADCT_RECON_F32 ? ADCT_INVT(OUT_I16, REC_F32) : ADCT_INVT(OUT_I16, REC_U8);
    if (coef_t == ADCT_COEF_I32) return dst_t == ADCT_RECON_F32 ? ADCT_INVT(OUT_I32, REC_F32) : ADCT_INVT(OUT_I32, REC_U8);
    return dst_t == ADCT_RECON_F32 ? ADCT_INVT(OUT_F32, REC_F32) : ADCT_INVT(OUT_F32, REC_U8);
#undef ADCT_INVT
  }
  if (coef_t == ADCT_COEF_I16) {  // u8 planes with w % 16 != 0: TMA ring in, per-lane stores out
    CUtensorMap map;
    if ((st = make_i16_map(&map, coef, n, h, w, coef_pitch, coef_img_stride))) return st;
    return dst_t == ADCT_RECON_F32
               ? launch_tma_kernel(k_inverse_i16<REC_F32>, map, p, p.tiles, s0, 2, 2 * TILE_BYTES)
               : launch_tma_kernel(k_inverse_i16<REC_U8>, map, p, p.tiles, s0, 2, 2 * TILE_BYTES);
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (int64_t)sms * 3;
  const int64_t need = (p.tiles + WARPS - 1) / WARPS;
  if (grid > need) grid = need;
  cudaStream_t s = (cudaStream_t)stream;
#define ADCT_INV(IN, RC) k_inverse<IN, RC><<<(unsigned)grid, WARPS * 32, 0, s>>>(p)
  if (coef_t == ADCT_COEF_I16) {
    if (dst_t == ADCT_RECON_F32) ADCT_INV(OUT_I16, REC_F32); else ADCT_INV(OUT_I16, REC_U8);
  } else if (coef_t == ADCT_COEF_I32) {
    if (dst_t == ADCT_RECON_F32) ADCT_INV(OUT_I32, REC_F32); else ADCT_INV(OUT_I32, REC_U8);
  } else {
    if (dst_t == ADCT_RECON_F32) ADCT_INV(OUT_F32, REC_F32); else ADCT_INV(OUT_F32, REC_U8);
  }
#undef ADCT_INV
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e);
}

adct_status adct_compress_psnr(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                               int64_t img_stride, int r, float q, void* recon, adct_recon_t recon_t,
                               int64_t recon_pitch, int64_t recon_img_stride, double* sse,
                               adct_stream_t stream) {
  adct_status st = check_geom(n, h, w);
  if (st) return st;
  if (r < 1 || r > 64 || !(q >= 0.f) || isinf(q)) return ADCT_EINVAL;
  if (recon_t != ADCT_RECON_NONE && recon_t != ADCT_RECON_F32 && recon_t != ADCT_RECON_U8) return ADCT_EINVAL;
  if (!sse) return ADCT_EINVAL;
  if ((st = check_plane(src, h, w, pitch, img_stride))) return st;
  if ((uintptr_t)sse & 7u) return ADCT_EALIGN;
  if (recon_t != ADCT_RECON_NONE &&
      (st = check_plane(recon, h, w * (recon_t == ADCT_RECON_F32 ? 4 : 1), recon_pitch, recon_img_stride)))
    return st;
  CUtensorMap map;
  if ((st = make_u8_map(&map, src, n, h, w, pitch, img_stride))) return st;
#ifndef ADCT_RECON_TMA_STORE
#define ADCT_RECON_TMA_STORE 1
#endif
  // reconstruction through shared-memory staging + TMA bulk stores (u8: only for w % 16 == 0, a
  // bulk store writes a row's last partial 16-byte chunk whole)
  const bool bulk = ADCT_RECON_TMA_STORE && (recon_t == ADCT_RECON_F32 || (recon_t == ADCT_RECON_U8 && (w & 15) == 0));
  CUtensorMap omap;
  memset(&omap, 0, sizeof(omap));
  if (bulk) {
    st = recon_t == ADCT_RECON_F32
             ? make_plane_map(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, recon, n, h, w, recon_pitch, recon_img_stride)
             : make_u8_map(&omap, (const uint8_t*)recon, n, h, w, recon_pitch, recon_img_stride);
    if (st) return st;
  }
  CompressParams p;
  memset(&p, 0, sizeof(p));
  p.h16magic = 0x64646464u;
  p.geo = make_geo(h, w);
  p.tiles = p.geo.per_img * n;
  p.h = (int)h;
  p.w = (int)w;
  p.sse = sse;
  p.recon = (uint8_t*)recon;
  p.recon_pitch = recon_pitch;
  p.recon_img_stride = recon_img_stride;
  const int fxk = fx_exponent(h * w, FX_BOUND_SSE);
  p.fx_scale = ldexp(1.0, fxk);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(sse, 0, sizeof(double) * (size_t)n, s);
  if (e != cudaSuccess) return cuda_fail(e);
  if ((st = compress_dispatch(map, omap, bulk, p, r, q, recon_t, s))) return st;
  return fx_finish(sse, n, fxk, s);
}

adct_status adct_compress_sse576(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                                 int64_t img_stride, int r, uint64_t* sse576, double* sse,
                                 adct_stream_t stream) {
  adct_status st = check_geom(n, h, w);
  if (st) return st;
  if (r < 1 || r > 64 || !sse576) return ADCT_EINVAL;
  if (h * w > (int64_t(1) << 26)) return ADCT_EINVAL;  // per-image sum < 2^63 (|576 x - R| <= 329205)
  if ((st = check_plane(src, h, w, pitch, img_stride))) return st;
  if (((uintptr_t)sse576 & 7u) || ((uintptr_t)sse & 7u)) return ADCT_EALIGN;
  CUtensorMap map;
  if ((st = make_u8_map(&map, src, n, h, w, pitch, img_stride))) return st;
  CompressParams p;
  memset(&p, 0, sizeof(p));
  p.geo = make_geo(h, w);
  p.tiles = p.geo.per_img * n;
  p.h = (int)h;
  p.w = (int)w;
  p.sse576 = reinterpret_cast<unsigned long long*>(sse576);
  p.h16magic = 0x64646464u;  // f16 pixel pairs of the error route (k_compress_exact)
  fill_zonal_tables(p.tab, r);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(sse576, 0, sizeof(uint64_t) * (size_t)n, s);
  if (e != cudaSuccess) return cuda_fail(e);
  CompressKernel ek = exact_kernel(r);  // C5's r: compile-time mask; other r: the runtime mask
  if ((st = launch_compress(ek ? ek : &k_compress_exact<2>, RT, map, p, s))) return st;
  if (!sse) return ADCT_OK;
  const int64_t blocks = (n + 255) / 256;
  k_sse576_to_f64<0><<<(unsigned)(blocks < 1024 ? blocks : 1024), 256, 0, s>>>(p.sse576, sse, n);
  ++g_launches;
  e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e);
}

// Symmetric 8x8 eigendecomposition by cyclic Jacobi rotations (host, double): A = V diag(w) V^T.
static void jacobi8(const double* Ain, double* w, double* V) {
  double A[64];
  for (int i = 0; i < 64; ++i) {
    A[i] = Ain[i];
    V[i] = (i % 9 == 0) ? 1.0 : 0.0;
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < 8; ++i)
      for (int j = i + 1; j < 8; ++j) off += A[i * 8 + j] * A[i * 8 + j];
    if (off < 1e-30) break;
    for (int p = 0; p < 8; ++p)
      for (int q = p + 1; q < 8; ++q) {
        const double apq = A[p * 8 + q];
        if (fabs(apq) < 1e-300) continue;
        const double th = (A[q * 8 + q] - A[p * 8 + p]) / (2.0 * apq);
        const double tt = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), sn = tt * c;
        for (int k = 0; k < 8; ++k) {  // A <- J^T A J
          const double akp = A[k * 8 + p], akq = A[k * 8 + q];
          A[k * 8 + p] = c * akp - sn * akq;
          A[k * 8 + q] = sn * akp + c * akq;
        }
        for (int k = 0; k < 8; ++k) {
          const double apk = A[p * 8 + k], aqk = A[q * 8 + k];
          A[p * 8 + k] = c * apk - sn * aqk;
          A[q * 8 + k] = sn * apk + c * aqk;
        }
        for (int k = 0; k < 8; ++k) {
          const double vkp = V[k * 8 + p], vkq = V[k * 8 + q];
          V[k * 8 + p] = c * vkp - sn * vkq;
          V[k * 8 + q] = sn * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < 8; ++i) w[i] = A[i * 9];
}

// Orthogonal polar factor (T T^T)^(-1/2) T of an invertible T (F4 for ceil(2C)).
static bool polar_factor(const double* T, double* out) {
  double G[64], w[8], V[64], S[64];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double a = 0.0;
      for (int k = 0; k < 8; ++k) a += T[i * 8 + k] * T[j * 8 + k];
      G[i * 8 + j] = a;
    }
  jacobi8(G, w, V);
  for (int i = 0; i < 8; ++i)
    if (!(w[i] > 1e-12)) return false;  // singular (e.g. floor(2C): a zero row)
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double a = 0.0;
      for (int k = 0; k < 8; ++k) a += V[i * 8 + k] * V[j * 8 + k] / sqrt(w[k]);
      S[i * 8 + j] = a;
    }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double a = 0.0;
      for (int k = 0; k < 8; ++k) a += S[i * 8 + k] * T[k * 8 + j];
      out[i * 8 + j] = a;
    }
  return true;
}

// The library's own matrices (independent of the CPU oracle): exact DCT-II from cos, C0 = [2C]
// with Matlab rounding, S from diag(C0 C0^T)^(-1/2), SDCT = sign(C)/(2 sqrt 2), coarse = C0 / 2,
// ceil variant = polar factor of ceil(2C) (F4).
static void build_matrix(adct_transform_t t, double* M) {
  if (t == ADCT_T_CEIL) {
    double T[64];
    for (int m = 0; m < 8; ++m)
      for (int n = 0; n < 8; ++n)
        T[m * 8 + n] = ceil(2.0 * (m == 0 ? 1.0 / (2.0 * sqrt(2.0)) : 0.5) * cos((2 * n + 1) * m * 3.14159265358979323846 / 16.0));
    polar_factor(T, M);  // ceil(2C) is invertible (det 16)
    return;
  }
  const double PI = 3.14159265358979323846;
  double C[64];
  for (int m = 0; m < 8; ++m)
    for (int n = 0; n < 8; ++n)
      C[m * 8 + n] = (m == 0 ? 1.0 / (2.0 * sqrt(2.0)) : 0.5) * cos((2 * n + 1) * m * PI / 16.0);
  for (int i = 0; i < 64; ++i) {
    const double twoc = 2.0 * C[i];
    const double c0 = (twoc < 0 ? -1.0 : 1.0) * floor(fabs(twoc) + 0.5);  // round half away from zero
    const double sgn = (C[i] > 1e-12) ? 1.0 : (C[i] < -1e-12 ? -1.0 : 0.0);
    switch (t) {
      case ADCT_T_DCT: M[i] = C[i]; break;
      case ADCT_T_SDCT: M[i] = sgn / (2.0 * sqrt(2.0)); break;
      case ADCT_T_COARSE: M[i] = 0.5 * c0; break;
      default: M[i] = c0; break;  // PROPOSED: scaled below
    }
  }
  if (t == ADCT_T_PROPOSED) {
    for (int m = 0; m < 8; ++m) {
      double d = 0.0;
      for (int n = 0; n < 8; ++n) d += M[m * 8 + n] * M[m * 8 + n];
      for (int n = 0; n < 8; ++n) M[m * 8 + n] /= sqrt(d);
    }
  }
}

adct_status adct_transform_matrix(adct_transform_t t, double* out) {
  if (!out || t < ADCT_T_PROPOSED || t == ADCT_T_CUSTOM || t > ADCT_T_CEIL) return ADCT_EINVAL;
  build_matrix(t, out);
  return ADCT_OK;
}

adct_status adct_compress_psnr_dense(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                                     int64_t img_stride, int r, adct_transform_t t, const double* custom,
                                     float* recon, int64_t recon_pitch, int64_t recon_img_stride,
                                     double* sse, adct_stream_t stream) {
  adct_status st = check_geom(n, h, w);
  if (st) return st;
  if (r < 1 || r > 64 || !sse) return ADCT_EINVAL;
  if (t < ADCT_T_PROPOSED || t > ADCT_T_CEIL || (t == ADCT_T_CUSTOM && !custom)) return ADCT_EINVAL;
  if ((st = check_plane(src, h, w, pitch, img_stride))) return st;
  if (recon && (st = check_plane(recon, h, w * 4, recon_pitch, recon_img_stride))) return st;
  if ((uintptr_t)sse & 7u) return ADCT_EALIGN;
  CUtensorMap map;
  if ((st = make_u8_map(&map, src, n, h, w, pitch, img_stride))) return st;
  DenseParams p;
  memset(&p, 0, sizeof(p));
  p.geo = make_geo(h, w);
  p.tiles = p.geo.per_img * n;
  p.h = (int)h;
  p.w = (int)w;
  p.sse = sse;
  p.recon = recon;
  p.recon_pitch = recon_pitch;
  p.recon_img_stride = recon_img_stride;
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l)
      if (zz_host(k, l) < r) p.keep_raster |= 1ull << (k * 8 + l);
  double Tm[64];
  if (t == ADCT_T_CUSTOM) {
    for (int i = 0; i < 64; ++i) {
      if (!isfinite(custom[i])) return ADCT_EINVAL;
      Tm[i] = custom[i];
    }
  } else {
    build_matrix(t, Tm);
  }
  for (int i = 0; i < 64; ++i) p.T[i] = (float)Tm[i];
  // a caller matrix need not be orthogonal: |x^_ij| <= 255 (max_i sum_k |T_ki| s_k)^2 with
  // s_k = sum_m |T_km| bounds every reconstructed pixel, so the per-pixel squared error is below
  // (255 + that)^2 (fixed-point range of the deterministic SSE)
  double colmax = 0.0;
  for (int i = 0; i < 8; ++i) {
    double c = 0.0;
    for (int k = 0; k < 8; ++k) {
      double sk = 0.0;
      for (int m = 0; m < 8; ++m) sk += fabs(Tm[k * 8 + m]);
      c += fabs(Tm[k * 8 + i]) * sk;
    }
    colmax = fmax(colmax, c);
  }
  const double emax = 255.0 * (1.0 + colmax * colmax) + 1.0;
  int bl = 0;
  while (ldexp(1.0, bl) < emax * emax && bl < 120) ++bl;
  const int fxk = fx_exponent(h * w, bl);
  p.fx_scale = ldexp(1.0, fxk);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(sse, 0, sizeof(double) * (size_t)n, s);
  if (e != cudaSuccess) return cuda_fail(e);
  if ((st = launch_tma_kernel(k_compress_dense<0>, map, p, p.tiles, s))) return st;
  return fx_finish(sse, n, fxk, s);
}

adct_status adct_compress_psnr_sdct(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                                    int64_t img_stride, int r, double* sse, adct_stream_t stream) {
  adct_status st = check_geom(n, h, w);
  if (st) return st;
  if (r < 1 || r > 64 || !sse) return ADCT_EINVAL;
  if ((st = check_plane(src, h, w, pitch, img_stride))) return st;
  if ((uintptr_t)sse & 7u) return ADCT_EALIGN;
  CUtensorMap map;
  if ((st = make_u8_map(&map, src, n, h, w, pitch, img_stride))) return st;
  CompressParams p;
  memset(&p, 0, sizeof(p));
  p.h16magic = 0x64646464u;
  p.geo = make_geo(h, w);
  p.tiles = p.geo.per_img * n;
  p.h = (int)h;
  p.w = (int)w;
  p.sse = sse;
  fill_bfly_pairs(p.tab);
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l) {
      const float m = zz_host(k, l) < r ? 1.f : 0.f;  // M_r as 0 / 1 weights (Z = Y / 8 folded in the 1/64)
      p.tab.w[k * 8 + l] = make_float2(m, m);
      p.tab.c[k * 8 + l] = make_float2(-KF * m, -KF * m);
    }
  // the SDCT is not orthogonal: |x^| <= |R| / 64 <= 64 * 16320 / 64, so (x - x^)^2 < 2^28 per pixel
  const int fxk = fx_exponent(h * w, 28);
  p.fx_scale = ldexp(1.0, fxk);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(sse, 0, sizeof(double) * (size_t)n, s);
  if (e != cudaSuccess) return cuda_fail(e);
  if ((st = launch_tma_kernel(k_compress_sdct<0>, map, p, p.tiles, s, 2))) return st;
  return fx_finish(sse, n, fxk, s);
}

}  // extern "C"
namespace {
// anti-diagonal energies of every image; SMAX = 14 (all) or 7 (r <= 36: slots 8..14 = UINT64_MAX)
adct_status diag_energy_impl(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch, int64_t img_stride,
                             int smax, uint64_t* energy, cudaStream_t s) {
  adct_status st = check_geom(n, h, w);
  if (st) return st;
  if (!energy) return ADCT_EINVAL;
  if ((st = check_plane(src, h, w, pitch, img_stride))) return st;
  if ((uintptr_t)energy & 7u) return ADCT_EALIGN;
  CUtensorMap map;
  if ((st = make_u8_map(&map, src, n, h, w, pitch, img_stride))) return st;
  DiagParams p;
  memset(&p, 0, sizeof(p));
  p.geo = make_geo(h, w);
  p.tiles = p.geo.per_img * n;
  p.h = (int)h;
  p.w = (int)w;
  p.energy = reinterpret_cast<unsigned long long*>(energy);
  cudaError_t e = cudaMemsetAsync(energy, 0, sizeof(uint64_t) * 16 * (size_t)n, s);
  if (e == cudaSuccess && smax < 14)  // not computed: UINT64_MAX (adct_sweep_psnr answers NaN)
    e = cudaMemset2DAsync(energy + smax + 1, 16 * sizeof(uint64_t), 0xFF, (14 - smax) * sizeof(uint64_t),
                          (size_t)n, s);
  if (e != cudaSuccess) return cuda_fail(e);
  return smax == 14 ? launch_tma_kernel(k_diag_energy<14>, map, p, p.tiles, s, DIAG_ST)
                    : launch_tma_kernel(k_diag_energy<7>, map, p, p.tiles, s, DIAG_ST);
}
}  // namespace
extern "C" {

adct_status adct_diag_energy(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch, int64_t img_stride,
                             uint64_t* energy, adct_stream_t stream) {
  return diag_energy_impl(src, n, h, w, pitch, img_stride, 14, energy, (cudaStream_t)stream);
}

adct_status adct_diag_energy_prefix(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                                    int64_t img_stride, int r_max, uint64_t* energy, adct_stream_t stream) {
  if (r_max < 1 || r_max > 64) return ADCT_EINVAL;
  return diag_energy_impl(src, n, h, w, pitch, img_stride, r_max <= 36 ? 7 : 14, energy, (cudaStream_t)stream);
}

adct_status adct_sweep_psnr(const uint64_t* energy, int64_t n, int64_t pixels, const int* r_list, int n_r, double* sse,
                            double* psnr, adct_stream_t stream) {
  if (!energy || !r_list || !sse || !psnr || n < 1 || pixels < 1 || n_r < 1 || n_r > 16) return ADCT_EINVAL;
  if (((uintptr_t)energy & 7u) || ((uintptr_t)sse & 7u) || ((uintptr_t)psnr & 7u)) return ADCT_EALIGN;
  SweepList L;
  memset(&L, 0, sizeof(L));
  L.n_r = n_r;
  for (int k = 0; k < n_r; ++k) {
    int s = -1;
    for (int d = 0; d < 15; ++d) {  // r = number of positions with k + l <= d
      const int rd = d <= 7 ? (d + 1) * (d + 2) / 2 : 64 - (14 - d) * (15 - d) / 2;
      if (rd == r_list[k]) s = d;
    }
    if (s < 0) return ADCT_EINVAL;  // only full anti-diagonal r: 1,3,6,10,15,21,28,36,43,49,54,58,61,63,64
    L.diag[k] = s;
  }
  const int64_t total = n * n_r;
  k_sweep_psnr<0><<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const unsigned long long*>(energy), n, L, (double)pixels, sse, psnr);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e);
}

adct_status adct_uqi(const uint8_t* x, int64_t n, int64_t h, int64_t w, int64_t x_pitch, int64_t x_img_stride,
                     const float* y, int64_t y_pitch, int64_t y_img_stride, double* uqi, adct_stream_t stream) {
  adct_status st = check_geom(n, h, w);
  if (st) return st;
  if (!x || !y || !uqi) return ADCT_EINVAL;
  if (x_pitch < w || x_img_stride < h * x_pitch || y_pitch < 4 * w || y_img_stride < h * y_pitch) return ADCT_EINVAL;
  if (((uintptr_t)y & 3u) || (y_pitch & 3) || (y_img_stride & 3) || ((uintptr_t)uqi & 7u)) return ADCT_EALIGN;
  if (n > 65535) return ADCT_EINVAL;
  UqiParams p;
  memset(&p, 0, sizeof(p));
  p.x = x;
  p.x_pitch = x_pitch;
  p.x_img_stride = x_img_stride;
  p.y = y;
  p.y_pitch = y_pitch;
  p.y_img_stride = y_img_stride;
  p.h = (int)h;
  p.w = (int)w;
  p.tiles_x = (int)((w - 7 + UQI_T - 1) / UQI_T);
  p.tiles_y = (int)((h - 7 + UQI_T - 1) / UQI_T);
  p.inv_windows = 1.0 / ((double)(h - 7) * (double)(w - 7));
  p.out = uqi;
  // the mean UQI lies in [-1, 1]: a 2^-52 fixed-point grid (deterministic CTA partial sums)
  constexpr int kUqiFx = 52;
  p.fx_scale = ldexp(1.0, kUqiFx);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(uqi, 0, sizeof(double) * (size_t)n, s);
  if (e != cudaSuccess) return cuda_fail(e);
  k_uqi<0><<<dim3(p.tiles_x, p.tiles_y, (unsigned)n), 256, 0, s>>>(p);
  ++g_launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e);
  return fx_finish(uqi, n, kUqiFx, s);
}

adct_status adct_quant_reciprocals(float q, float* c_out) {
  if (!c_out || !(q > 0.f) || isinf(q)) return ADCT_EINVAL;
  for (int k = 0; k < 8; ++k)
    for (int l = 0; l < 8; ++l) c_out[k * 8 + l] = quant_recip(q, dval(k) * dval(l));
  return ADCT_OK;
}

adct_status adct_psnr(const double* sse, int64_t count, int64_t pixels, double* psnr, adct_stream_t stream) {
  if (!sse || !psnr || count < 1 || pixels < 1) return ADCT_EINVAL;
  if (((uintptr_t)sse & 7u) || ((uintptr_t)psnr & 7u)) return ADCT_EALIGN;
  const int64_t blocks = (count + 255) / 256;
  k_psnr<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(sse, count, (double)pixels, psnr);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ADCT_OK : cuda_fail(e);
}

}  // extern "C"

namespace {
// adct_compress_psnr_multi with the per-r rows `sse_stride` doubles apart (the host entry writes
// chunks of images into columns of its [n_r][n] buffer).  Validation done by the callers.
adct_status compress_multi_strided(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                                   int64_t img_stride, const int* r_list, int n_r, double* sse, int64_t sse_stride,
                                   cudaStream_t s) {
  // the compiled set (BASELINE C5's r, any order, each once) -> one fused kernel
  int rowmap[8];
  bool fused = (n_r == RSetC5::n);
  for (int k = 0; fused && k < RSetC5::n; ++k) {
    int hit = -1;
    for (int i = 0; i < n_r; ++i)
      if (r_list[i] == RSetC5::r[k]) hit = (hit < 0) ? i : -2;
    fused = hit >= 0;
    rowmap[k] = hit;
  }
  adct_status st = ADCT_OK;
  if (!fused) {  // any other set: independent passes
    for (int k = 0; k < n_r; ++k)
      if ((st = adct_compress_psnr(src, n, h, w, pitch, img_stride, r_list[k], 0.f, nullptr, ADCT_RECON_NONE, 0, 0,
                                   sse + (int64_t)k * sse_stride, s)))
        return st;
    return ADCT_OK;
  }
  CUtensorMap map;
  if ((st = make_u8_map(&map, src, n, h, w, pitch, img_stride))) return st;
  CompressParams p;
  memset(&p, 0, sizeof(p));
  p.h16magic = 0x64646464u;
  p.geo = make_geo(h, w);
  p.tiles = p.geo.per_img * n;
  p.h = (int)h;
  p.w = (int)w;
  p.sse = sse;
  p.sse_stride = sse_stride;
  for (int k = 0; k < 8; ++k) p.rowmap[k] = rowmap[k];
  fill_zonal_tables(p.tab, 64);  // per-class weights (the compile-time masks need nothing else)
  const int fxk = fx_exponent(h * w, FX_BOUND_SSE);
  p.fx_scale = ldexp(1.0, fxk);
  cudaError_t e = sse_stride == n ? cudaMemsetAsync(sse, 0, sizeof(double) * (size_t)(n * n_r), s)
                                  : cudaMemset2DAsync(sse, sizeof(double) * (size_t)sse_stride, 0,
                                                      sizeof(double) * (size_t)n, (size_t)n_r, s);
  if (e != cudaSuccess) return cuda_fail(e);
#ifndef ADCT_SWEEP_INC
#define ADCT_SWEEP_INC 1
#endif
  if (ADCT_SWEEP_INC) {  // incremental: band b = anti-diagonal b completes r = (b + 1)(b + 2) / 2
    for (int b = 0; b < 8; ++b) p.rowmap[b] = rowmap[7 - b];  // RSetC5 lists r = 36, 28, ..., 1
    st = launch_compress(sweep_inc_kernel_c5(), 1, map, p, s);
  } else {
    st = launch_compress(multi_kernel_c5(), 1, map, p, s);
  }
  if (st) return st;
  for (int k = 0; k < n_r && st == ADCT_OK; ++k) st = fx_finish(sse + (int64_t)k * sse_stride, n, fxk, s);
  return st;
}
}  // namespace

extern "C" {

adct_status adct_compress_psnr_multi(const uint8_t* src, int64_t n, int64_t h, int64_t w, int64_t pitch,
                                     int64_t img_stride, const int* r_list, int n_r, double* sse,
                                     adct_stream_t stream) {
  adct_status st = check_geom(n, h, w);
  if (st) return st;
  if (!r_list || n_r < 1 || n_r > 64 || !sse) return ADCT_EINVAL;
  for (int k = 0; k < n_r; ++k)
    if (r_list[k] < 1 || r_list[k] > 64) return ADCT_EINVAL;
  if ((st = check_plane(src, h, w, pitch, img_stride))) return st;
  if ((uintptr_t)sse & 7u) return ADCT_EALIGN;
  return compress_multi_strided(src, n, h, w, pitch, img_stride, r_list, n_r, sse, n, (cudaStream_t)stream);
}

adct_status adct_compress_psnr_host(const uint8_t* host_src, int64_t n, int64_t h, int64_t w,
                                    int64_t host_pitch, int64_t host_img_stride, const int* r_list, int n_r,
                                    float q, uint8_t* dev_buf, int64_t dev_buf_bytes, double* dev_sse,
                                    double* host_psnr, adct_stream_t stream, adct_stream_t copy_stream) {
  adct_status st = check_geom(n, h, w);
  if (st) return st;
  if (!host_src || !r_list || n_r < 1 || n_r > 64 || !dev_buf || !dev_sse || !host_psnr) return ADCT_EINVAL;
  if (host_pitch < w || host_img_stride < h * host_pitch) return ADCT_EINVAL;
  for (int k = 0; k < n_r; ++k)
    if (r_list[k] < 1 || r_list[k] > 64) return ADCT_EINVAL;
  if (!(q >= 0.f) || isinf(q)) return ADCT_EINVAL;
  const int64_t dpitch = (w + 15) & ~(int64_t)15;
  const int64_t dimg = dpitch * h;
  if (!aligned16(dev_buf) || ((uintptr_t)dev_sse & 7u)) return ADCT_EALIGN;
  const int64_t cap = dev_buf_bytes / dimg;  // images the staging buffer holds
  if (cap < 1) return ADCT_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  auto stage = [&](uint8_t* dst, int64_t i0, int64_t m, cudaStream_t cs) -> cudaError_t {
    if (host_img_stride == h * host_pitch && host_pitch == dpitch)
      return cudaMemcpyAsync(dst, host_src + i0 * host_img_stride, (size_t)(m * dimg), cudaMemcpyHostToDevice, cs);
    cudaError_t e = cudaSuccess;
    for (int64_t j = 0; j < m && e == cudaSuccess; ++j)
      e = cudaMemcpy2DAsync(dst + j * dimg, (size_t)dpitch, host_src + (i0 + j) * host_img_stride,
                            (size_t)host_pitch, (size_t)w, (size_t)h, cudaMemcpyHostToDevice, cs);
    return e;
  };
  // zonal passes: the fused multi-r kernel when the set is BASELINE C5's (one read, one forward per
  // tile for all r), independent passes otherwise; the quantiser: one pass per r
  auto compress_chunk = [&](const uint8_t* buf, int64_t i0, int64_t m) -> adct_status {
    if (q == 0.f) return compress_multi_strided(buf, m, h, w, dpitch, dimg, r_list, n_r, dev_sse + i0, n, s);
    for (int k = 0; k < n_r; ++k) {
      adct_status st2 = adct_compress_psnr(buf, m, h, w, dpitch, dimg, r_list[k], q, nullptr, ADCT_RECON_NONE, 0,
                                           0, dev_sse + (int64_t)k * n + i0, stream);
      if (st2) return st2;
    }
    return ADCT_OK;
  };
  const int64_t half = cap / 2;
  cudaStream_t cs = (cudaStream_t)copy_stream;
  if (cs && cs != s && n >= 2 && half >= 1) {
    // Double-buffered pipeline on the caller's copy stream: the host->device copy of chunk c+1
    // overlaps the passes of chunk c.  Chunks of about n/8 images, two per buffer; ordering by
    // events (cheap to create; no stream is created), so the whole call can also be captured into
    // a CUDA graph (fork / join through the events).
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(half, (n + 7) / 8));
    cudaEvent_t ready[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr}, start = nullptr;
    cudaError_t e = cudaSuccess;
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
      e = cudaEventCreateWithFlags(&ready[b], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&freed[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    // the staging buffer may still be read by work already queued on the caller's stream
    if (e == cudaSuccess) e = cudaEventRecord(start, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, start, 0);
    adct_status st2 = ADCT_OK;
    int64_t c = 0;
    for (int64_t i0 = 0; i0 < n && e == cudaSuccess && st2 == ADCT_OK; i0 += chunk, ++c) {
      const int b = (int)(c & 1);
      const int64_t m = std::min<int64_t>(chunk, n - i0);
      uint8_t* buf = dev_buf + b * chunk * dimg;
      if (c >= 2) e = cudaStreamWaitEvent(cs, freed[b], 0);  // chunk c-2's passes are done with buf
      if (e == cudaSuccess) e = stage(buf, i0, m, cs);
      if (e == cudaSuccess) e = cudaEventRecord(ready[b], cs);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ready[b], 0);
      if (e == cudaSuccess) st2 = compress_chunk(buf, i0, m);
      if (e == cudaSuccess && st2 == ADCT_OK) e = cudaEventRecord(freed[b], s);
    }
    // events are released once their pending work completes (no host synchronisation)
    for (int b = 0; b < 2; ++b) {
      if (ready[b]) cudaEventDestroy(ready[b]);
      if (freed[b]) cudaEventDestroy(freed[b]);
    }
    if (start) cudaEventDestroy(start);
    if (e != cudaSuccess) return cuda_fail(e);
    if (st2) return st2;
  } else {  // copies and passes alternate on the caller's stream
    for (int64_t i0 = 0; i0 < n; i0 += cap) {
      const int64_t m = std::min<int64_t>(cap, n - i0);
      cudaError_t e = stage(dev_buf, i0, m, s);
      if (e != cudaSuccess) return cuda_fail(e);
      if ((st = compress_chunk(dev_buf, i0, m))) return st;
    }
  }
  // PSNR of every (r, image) into the second half of dev_sse, then one device->host copy
  double* dev_psnr = dev_sse + (int64_t)n_r * n;
  if ((st = adct_psnr(dev_sse, n * n_r, h * w, dev_psnr, stream))) return st;
  cudaError_t e = cudaMemcpyAsync(host_psnr, dev_psnr, sizeof(double) * (size_t)(n * n_r), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return cuda_fail(e);
  return ADCT_OK;
}

}  // extern "C"

namespace adct {
CompressKernel zonal_kernel_part0(int r);
CompressKernel zonal_kernel_part1(int r);
CompressKernel zonal_kernel_part2(int r);
CompressKernel zonal_kernel_part3(int r);
CompressKernel zonal_kernel(int r) {
  switch ((r - 1) / 16) {
    case 0: return zonal_kernel_part0(r);
    case 1: return zonal_kernel_part1(r);
    case 2: return zonal_kernel_part2(r);
    default: return zonal_kernel_part3(r);
  }
}
}  // namespace adct
