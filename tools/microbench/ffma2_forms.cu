// Throughput of the f32x2 operand forms used by the quantiser kernel (sm_100a):
// FFMA2 R, R, imm / FFMA2 R, R.F32 (scalar broadcast), R / FADD2 R, imm / FADD2 R, R, each over 8
// independent chains per thread, 8 warps x 148*8 CTAs.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_forms ffma2_forms.cu
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
#define CH 8
template <int OP>
__global__ void __launch_bounds__(256) kern(float2* out, float s, float t) {
  float2 r[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) r[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  const float2 sv = make_float2(s, s), tv = make_float2(t, t);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) r[c] = __ffma2_rn(r[c], make_float2(0.999f, 0.999f), make_float2(0.5f, 0.5f));  // R, imm, imm
      if (OP == 1) r[c] = __ffma2_rn(r[c], sv, r[(c + 1) % CH]);                                    // R, R.F32, R
      if (OP == 2) r[c] = __ffma2_rn(r[c], make_float2(0.999f, 0.999f), r[(c + 1) % CH]);           // R, imm, R
      if (OP == 3) r[c] = __fadd2_rn(r[c], make_float2(0.5f, 0.5f));                               // R, imm
      if (OP == 4) r[c] = __fadd2_rn(r[c], r[(c + 1) % CH]);                                        // R, R
      if (OP == 5) r[c] = __ffma2_rn(r[c], r[(c + 2) % CH], sv);                                    // R, R, R.F32
      if (OP == 6) r[c] = __ffma2_rn(r[c], r[(c + 2) % CH], r[(c + 1) % CH]);                       // 3 pairs
      if (OP == 7) r[c] = __fadd2_rn(r[c], tv);                                                     // R, R.F32
    }
  }
  float2 a = r[0];
#pragma unroll
  for (int c = 1; c < CH; ++c) a = __fadd2_rn(a, r[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
template <int OP>
void run(const char* name) {
  float2* out;
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(float2));
  kern<OP><<<148 * 8, 256>>>(out, 0.999f, 0.5f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<OP><<<148 * 8, 256>>>(out, 0.999f, 0.5f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double instr = 148.0 * 8 * 8 * ITERS * CH;  // warp instructions
  printf("%-28s %7.3f ms  %.3f warp-instr/ns/SM\n", name, ms, instr / (ms * 1e6) / 148);
  cudaFree(out);
}
int main() {
  run<0>("FFMA2 R, imm, imm");
  run<1>("FFMA2 R, R.F32 bcast, R");
  run<2>("FFMA2 R, imm, R");
  run<3>("FADD2 R, imm");
  run<4>("FADD2 R, R");
  run<5>("FFMA2 R, R, R.F32 bcast");
  run<6>("FFMA2 R, R, R (3 pairs)");
  run<7>("FADD2 R, R.F32 bcast");
  return 0;
}
