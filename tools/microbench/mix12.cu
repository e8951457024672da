// Achievable HBM rate for a 1 : 2 read : write stream (the C3 forward's traffic: 1 B/px of u8 in,
// 2 B/px of int16 out) with no transform: every thread widens 16 bytes to 16 int16 (one 128-bit
// load, two 128-bit stores), grid-stride, over the C3 batch (8192 x 512^2 = 2 GiB in, 4 GiB out);
// plus the 1 : 1 u8 copy for comparison with MEASURED_PEAKS.json's copy figure.  CUDA events,
// best of 10, several grid sizes (multiples of the 148 SMs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mix12 mix12.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) widen(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs(in + i);
    uint4 a, b;
    a.x = __byte_perm(v.x, 0, 0x4140); a.y = __byte_perm(v.x, 0, 0x4342);
    a.z = __byte_perm(v.y, 0, 0x4140); a.w = __byte_perm(v.y, 0, 0x4342);
    b.x = __byte_perm(v.z, 0, 0x4140); b.y = __byte_perm(v.z, 0, 0x4342);
    b.z = __byte_perm(v.w, 0, 0x4140); b.w = __byte_perm(v.w, 0, 0x4342);
    __stcs(out + 2 * i, a);
    __stcs(out + 2 * i + 1, b);
  }
}
__global__ void __launch_bounds__(256) copy8(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    __stcs(out + i, __ldcs(in + i));
}

int main() {
  const size_t px = (size_t)8192 * 512 * 512, n16 = px / 16;
  uint8_t* in;
  uint4* out;
  cudaMalloc(&in, px);
  cudaMalloc(&out, px * 2);
  cudaMemset(in, 7, px);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) {
    for (int per_sm : {4, 8, 16, 32}) {
      const int grid = 148 * per_sm;
      float best = 1e30f;
      for (int it = 0; it < 11; ++it) {
        cudaEventRecord(e0);
        if (mode == 0) widen<<<grid, 256>>>((const uint4*)in, out, n16);
        else copy8<<<grid, 256>>>((const uint4*)in, out, n16);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it) best = ms < best ? ms : best;
      }
      const double bytes = (double)px * (mode == 0 ? 3 : 2);
      printf("%-28s grid 148 x %2d: %.3f ms  %.1f GB/s\n", mode == 0 ? "widen u8 -> int16 (1:2)" : "copy u8 (1:1)", per_sm,
             best, bytes / (best * 1e-3) / 1e9);
    }
  }
  return cudaGetLastError() != cudaSuccess;
}
