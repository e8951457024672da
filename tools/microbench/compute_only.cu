// Compute-only throughput of the compress tile body (no TMA, no HBM): each warp runs
// compress_fwd + compress_inv on a tile staged once in shared memory, N times.  Reports the
// equivalent input bandwidth (4 KB per tile) so it can be compared with the HBM roofline.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -I../../include -I../../paper_1402_6034_b200/csrc -o compute_only compute_only.cu
#include <cstdio>
#include "adct_kernels.cuh"

using namespace adct;

template <int R, int MIN_CTAS>
__global__ void __launch_bounds__(128, MIN_CTAS) k_body(const uint8_t* src, CompressParams p, int iters, float* out) {
  __shared__ __align__(128) uint8_t tile[4][TILE_BYTES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4 * TILE_BYTES; i += blockDim.x) tile[0][i] = src[(blockIdx.x * 977 + i) % 65536];
  __syncthreads();
  float2 acc = f2(0.f);
  for (int it = 0; it < iters; ++it) {
    uint32_t Y[8][8];
    const uint8_t* t = tile[(warp + it) & 3];
    if constexpr (compress_resid_r(R)) {  // same per-r variant as k_compress
      compress_fwd<RESID + R, MODE_ZONAL>(t, lane, Y);
      acc = f2add(acc, compress_resid<R>(Y, p));
    } else {
      compress_fwd<R, MODE_ZONAL>(t, lane, Y);
      acc = f2add(acc, compress_inv<R, MODE_ZONAL, REC_NONE, compress_f16_rows(R)>(Y, t, lane, p, 0, 0, 0));
    }
  }
  if (acc.x == 1.2345f) out[0] = acc.y;
}

template <int R, int MIN_CTAS>
void run(const uint8_t* src, float* out, int sms, int dyn_smem = 0) {
  CompressParams p;
  memset(&p, 0, sizeof(p));
  p.h16magic = 0x64646464u;
  for (int k = 0; k < 64; ++k) {
    float w = (float)wval(k / 8, k % 8);
    p.tab.wc[wclass(k / 8, k % 8)] = w;
    p.tab.cc[wclass(k / 8, k % 8)] = -KF * w;
    p.tab.w[k] = make_float2(w, w);
    p.tab.c[k] = make_float2(-KF * w, -KF * w);
  }
  int occ = 0;
  cudaFuncSetAttribute(k_body<R, MIN_CTAS>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_body<R, MIN_CTAS>, 128, dyn_smem);
  int grid = sms * occ, iters = 2000;
  k_body<R, MIN_CTAS><<<grid, 128, dyn_smem>>>(src, p, 10, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_body<R, MIN_CTAS><<<grid, 128, dyn_smem>>>(src, p, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double tiles = (double)grid * 4 * iters;
  printf("r=%2d ctas/SM=%d: %.3f ms, %.0f GB/s-equivalent (%.3f of 6534), %.1f cycles/tile/SMSP @1.965GHz  %s\n", R, occ,
         ms, tiles * TILE_BYTES / ms / 1e6, tiles * TILE_BYTES / ms / 1e6 / 6534.1,
         ms * 1e-3 * 1.965e9 / (tiles / (sms * 4)), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* src;
  float* out;
  cudaMalloc(&src, 65536);
  cudaMalloc(&out, 64);
  uint8_t h[65536];
  for (int i = 0; i < 65536; ++i) h[i] = (uint8_t)((i * 2654435761u) >> 13);
  cudaMemcpy(src, h, 65536, cudaMemcpyHostToDevice);
  // at the library's per-r register cap (compress_minb), shared memory not limiting
  run<1, compress_minb(1)>(src, out, sms);
  run<3, compress_minb(3)>(src, out, sms);
  run<6, compress_minb(6)>(src, out, sms);
  run<10, compress_minb(10)>(src, out, sms);
  run<15, compress_minb(15)>(src, out, sms);
  run<21, compress_minb(21)>(src, out, sms);
  run<28, compress_minb(28)>(src, out, sms);
  run<36, compress_minb(36)>(src, out, sms);
  return 0;
}
