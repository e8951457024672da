// Pipe-throughput microbenchmark for the sm_100a instruction mix the ADCT kernels use.
// Measures lane-ops/clk/SM for IADD3, LOP3, PRMT, IMAD, FADD, FFMA, FADD2 (f32x2),
// FFMA2 and ALU/FMA mixes, plus the SM clock seen during the run.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

template <int OP>
__global__ void __launch_bounds__(256) kern(uint32_t* out, uint32_t seed, unsigned long long* clk) {
  uint32_t r[CH];
  unsigned long long rr[CH];
  uint32_t f[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    r[c] = seed * (threadIdx.x + 1 + c);
    f[c] = r[c] ^ 0x3f800000u;
    rr[c] = ((unsigned long long)r[c] << 32) | (r[c] ^ 0x3f800000u);
  }
  uint32_t k1 = seed ^ 0x1234u, k2 = seed ^ 0x4321u;
  unsigned long long kk = ((unsigned long long)k1 << 32) | k2;
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) asm volatile("add.s32 %0, %0, %1;" : "+r"(r[c]) : "r"(k1));
      if (OP == 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[c]) : "r"(k1), "r"(k2));
      if (OP == 2) asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(r[c]) : "r"(k1));
      if (OP == 3) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(k1), "r"(k2));
      if (OP == 4) asm volatile("add.f32 %0, %0, %1;" : "+r"(r[c]) : "r"(k1));
      if (OP == 5) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(k1), "r"(k2));
      if (OP == 6) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(rr[c]) : "l"(kk));
      if (OP == 7) asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(rr[c]) : "l"(kk));
      if (OP == 8) {  // IADD3 + FADD2 interleaved
        asm volatile("add.s32 %0, %0, %1;" : "+r"(r[c]) : "r"(k1));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(rr[c]) : "l"(kk));
      }
      if (OP == 9) {  // IADD3 + FADD interleaved
        asm volatile("add.s32 %0, %0, %1;" : "+r"(r[c]) : "r"(k1));
        asm volatile("add.f32 %0, %0, %1;" : "+r"(f[c]) : "r"(k1));
      }
      if (OP == 10) {  // 3-input integer add (IADD3 with three live operands)
        asm volatile("{.reg .s32 t; add.s32 t, %0, %1; add.s32 %0, t, %2;}" : "+r"(r[c]) : "r"(k1), "r"(k2));
      }
      if (OP == 11) asm volatile("mad.wide.s32 %0, %1, %1, %0;" : "+l"(rr[c]) : "r"(r[c]));
      if (OP == 12) asm volatile("add.f32 %0, %0, 0f3F800000;" : "+r"(r[c]));
      if (OP == 13) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3F800000;" : "+r"(r[c]));
      // live-operand variants: every source is a distinct, changing register
      if (OP == 14) asm volatile("{.reg .s32 t; add.s32 t, %0, %1; add.s32 %0, t, %2;}" : "+r"(r[c]) : "r"(r[(c + 1) % CH]), "r"(r[(c + 3) % CH]));
      if (OP == 15) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(rr[c]) : "l"(rr[(c + 1) % CH]), "l"(rr[(c + 3) % CH]));
      if (OP == 16) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(rr[c]) : "l"(rr[(c + 1) % CH]));
      if (OP == 17) asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(r[c]) : "r"(r[(c + 1) % CH]));
      if (OP == 18) {  // the compress mix: 3-input IADD3 + FADD2 + PRMT + FFMA2, all live operands
        asm volatile("{.reg .s32 t; add.s32 t, %0, %1; add.s32 %0, t, %2;}" : "+r"(r[c]) : "r"(r[(c + 1) % CH]), "r"(r[(c + 3) % CH]));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(rr[c]) : "l"(rr[(c + 1) % CH]));
        asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(f[c]) : "r"(r[(c + 2) % CH]));
        asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(rr[(c + 4) % CH]) : "l"(rr[(c + 5) % CH]), "l"(rr[(c + 6) % CH]));
      }
      // conversions: byte -> f32 (I2F.U8 with byte select), int -> f32 (I2FP), f16 -> f32 (HADD2.F32)
      if (OP == 19) asm volatile("{.reg .u32 t; shr.u32 t, %0, 8; cvt.rn.f32.u8 %0, t;}" : "+r"(r[c]));
      if (OP == 20) asm volatile("cvt.rn.f32.u32 %0, %0;" : "+r"(r[c]));
      if (OP == 21) asm volatile("{.reg .f16 h; mov.b32 {h, _}, %0; cvt.f32.f16 %0, h;}" : "+r"(r[c]));
      if (OP == 22) {  // PRMT + I2F.U8 interleaved: separate pipes?
        asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(r[c]) : "r"(k1));
        asm volatile("cvt.rn.f32.u8 %0, %0;" : "+r"(f[c]));
      }
      if (OP == 23) {  // FFMA2 + I2F.U8 interleaved
        asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(rr[c]) : "l"(kk));
        asm volatile("cvt.rn.f32.u8 %0, %0;" : "+r"(f[c]));
      }
      if (OP == 24) {  // PRMT + HADD2.F32 interleaved
        asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(r[c]) : "r"(k1));
        asm volatile("{.reg .f16 h; mov.b32 {h, _}, %0; cvt.f32.f16 %0, h;}" : "+r"(f[c]));
      }
      if (OP == 25) {  // FFMA2 + HADD2.F32 interleaved
        asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(rr[c]) : "l"(kk));
        asm volatile("{.reg .f16 h; mov.b32 {h, _}, %0; cvt.f32.f16 %0, h;}" : "+r"(f[c]));
      }
      if (OP == 26) {  // PRMT + I2FP.F32.U32 interleaved
        asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(r[c]) : "r"(k1));
        asm volatile("cvt.rn.f32.u32 %0, %0;" : "+r"(f[c]));
      }
      if (OP == 27) {  // FFMA2 + I2FP.F32.U32 interleaved
        asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(rr[c]) : "l"(kk));
        asm volatile("cvt.rn.f32.u32 %0, %0;" : "+r"(f[c]));
      }
      if (OP == 28) asm volatile("dp4a.u32.u32 %0, %0, %1, %0;" : "+r"(r[c]) : "r"(k1));
      if (OP == 29) {  // PRMT + IMAD interleaved (IMAD on the FMA pipe?)
        asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(r[c]) : "r"(k1));
        asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(f[c]) : "r"(k1), "r"(k2));
      }
      if (OP == 30) {  // FFMA2 + IMAD interleaved
        asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(rr[c]) : "l"(kk));
        asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(f[c]) : "r"(k1), "r"(k2));
      }
      // mixed-precision FMA: f16 x f16 + f32 -> f32 (SASS FHFMA)
      if (OP == 31) asm volatile("{.reg .f16 h; mov.b32 {h, _}, %1; fma.rn.f32.f16 %0, h, h, %0;}" : "+r"(r[c]) : "r"(k1));
      if (OP == 32) {  // FHFMA + FFMA2 interleaved
        asm volatile("{.reg .f16 h; mov.b32 {h, _}, %1; fma.rn.f32.f16 %0, h, h, %0;}" : "+r"(r[c]) : "r"(k1));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(rr[c]) : "l"(kk));
      }
      if (OP == 33) {  // FHFMA + PRMT interleaved
        asm volatile("{.reg .f16 h; mov.b32 {h, _}, %1; fma.rn.f32.f16 %0, h, h, %0;}" : "+r"(r[c]) : "r"(k1));
        asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(f[c]) : "r"(k2));
      }
      if (OP == 34) {  // FHFMA + FFMA (scalar) interleaved
        asm volatile("{.reg .f16 h; mov.b32 {h, _}, %1; fma.rn.f32.f16 %0, h, h, %0;}" : "+r"(r[c]) : "r"(k1));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(f[c]) : "r"(k1), "r"(k2));
      }
    }
  }
  unsigned long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= r[c] ^ f[c] ^ (uint32_t)rr[c] ^ (uint32_t)(rr[c] >> 32);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int OP>
void run(const char* name, int lanes_per_instr, int instr_per_chain_step, int sms) {
  uint32_t* out;
  unsigned long long* clk;
  cudaMalloc(&out, 148 * 64 * 256 * 4);
  cudaMalloc(&clk, 8);
  int blocks = sms * 8;
  kern<OP><<<blocks, 256>>>(out, 7, clk);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<OP><<<blocks, 256>>>(out, 7, clk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long cyc;
  cudaMemcpy(&cyc, clk, 8, cudaMemcpyDeviceToHost);
  double instrs = (double)blocks * 256 * ITERS * CH * instr_per_chain_step;
  double ghz = cyc / (ms * 1e6);  // block-0 cycles over wall time (approx SM clock)
  double lane_ops_per_clk_sm = instrs * lanes_per_instr / (ms * 1e-3) / (ghz * 1e9) / sms;
  printf("%-14s %8.3f ms  clk~%.3f GHz  warp-instr/clk/SM=%.2f  lane-ops/clk/SM=%.1f\n", name, ms, ghz,
         instrs / 32 / (ms * 1e-3) / (ghz * 1e9) / sms, lane_ops_per_clk_sm);
  cudaError_t e = cudaGetLastError();
  if (e) printf("err %s\n", cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs=%d\n", sms);
  run<0>("iadd", 1, 1, sms);
  run<10>("iadd3(2 ops)", 1, 2, sms);
  run<1>("lop3", 1, 1, sms);
  run<2>("prmt", 1, 1, sms);
  run<3>("imad", 1, 1, sms);
  run<11>("imad.wide", 1, 1, sms);
  run<4>("fadd", 1, 1, sms);
  run<12>("fadd-imm", 1, 1, sms);
  run<5>("ffma", 1, 1, sms);
  run<13>("ffma-imm", 1, 1, sms);
  run<6>("fadd2", 2, 1, sms);
  run<7>("ffma2", 2, 1, sms);
  run<8>("iadd+fadd2", 1, 2, sms);
  run<9>("iadd+fadd", 1, 2, sms);
  run<14>("iadd3 live", 1, 1, sms);
  run<15>("ffma2 live", 2, 1, sms);
  run<16>("fadd2 live", 2, 1, sms);
  run<17>("prmt live", 1, 1, sms);
  run<18>("mix4 live", 1, 4, sms);
  run<19>("i2f.u8(+shf)", 1, 2, sms);
  run<20>("i2fp.u32", 1, 1, sms);
  run<21>("hadd2.f32", 1, 1, sms);
  run<22>("prmt+i2f.u8", 1, 2, sms);
  run<23>("ffma2+i2f.u8", 1, 2, sms);
  run<24>("prmt+hadd2.f32", 1, 2, sms);
  run<25>("ffma2+hadd2.f32", 1, 2, sms);
  run<26>("prmt+i2fp", 1, 2, sms);
  run<27>("ffma2+i2fp", 1, 2, sms);
  run<28>("dp4a", 1, 1, sms);
  run<29>("prmt+imad", 1, 2, sms);
  run<30>("ffma2+imad", 1, 2, sms);
  run<31>("fhfma(f16*f16+f32)", 1, 1, sms);
  run<32>("fhfma+ffma2", 1, 2, sms);
  run<33>("fhfma+prmt", 1, 2, sms);
  run<34>("fhfma+ffma", 1, 2, sms);
  return 0;
}
