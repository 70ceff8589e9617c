// Issue/pipe microbenchmark (sm_100a): warp-instructions per clock per SMSP
// of single ops and 1:1 mixes, to tell which integer ops share the ALU pipe
// (rt 2 cycles/SMSP) and which go to the FMA pipe.  8 independent chains per
// thread, 32 warps per SM; check the SASS with cuobjdump -sass.
#include <cstdio>
#include <cuda_runtime.h>
#define CH 8
#define IT 256
template <int OP>
__global__ void __launch_bounds__(1024) k(unsigned *out, unsigned s0, unsigned s1) {
  unsigned x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x * (c + 3) ^ s0; y[c] = threadIdx.x + c * s1; }
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0 || OP == 2 || OP == 3 || OP == 5) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y[c]), "r"(s0));
      if (OP == 1 || OP == 2) asm volatile("add.u32 %0, %0, 7;" : "+r"(y[c]));
      if (OP == 3 || OP == 4) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y[c]) : "r"(s1), "r"(x[c]));
      if (OP == 5 || OP == 6) asm volatile("{.reg .pred p; setp.lt.u32 p, %0, %1; selp.u32 %0, %0, %1, p;}" : "+r"(y[c]) : "r"(s1));
      if (OP == 7 || OP == 8) asm volatile("popc.b32 %0, %0;" : "+r"(y[c]));
      if (OP == 8) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(s1), "r"(y[c]));
      if (OP == 9) asm volatile("add.u32 %0, %0, %1;" : "+r"(y[c]) : "r"(x[c]));
      if (OP == 10) asm volatile("shl.b32 %0, %0, %1;" : "+r"(y[c]) : "r"(x[c]));
      if (OP == 11) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(y[c]) : "r"(s1));
      if (OP == 13 || OP == 14 || OP == 15) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(y[c]), "r"(s0));
      if (OP == 13) asm volatile("shl.b32 %0, %0, %1;" : "+r"(y[c]) : "r"(x[c]));
      if (OP == 14) asm volatile("{.reg .pred p; setp.lt.u32 p, %0, %1; selp.u32 %0, %1, %2, p;}" : "+r"(y[c]) : "r"(x[c]), "r"(s1));
      if (OP == 15) asm volatile("{.reg .pred p; setp.lt.u32 p, %0, %1; @p add.u32 %0, %0, 3;}" : "+r"(y[c]) : "r"(x[c]));
      if (OP == 12) asm volatile("{.reg .pred p; setp.lt.u32 p, %0, %1; @p add.u32 %0, %0, 3;}" : "+r"(y[c]) : "r"(s1));
    }
  }
  unsigned r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) r ^= x[c] ^ y[c];
  if (r == 0x12345678u) out[0] = r;
}
template <int OP>
void run(const char *name, int n_inst, unsigned *o, int sms, int clk_khz) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<OP><<<sms * 2, 1024>>>(o, 1, 3);
  cudaEventRecord(a);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) k<OP><<<sms * 2, 1024>>>(o, 1, 3);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double warp_inst = (double)reps * sms * 2 * 32 * IT * CH * n_inst;
  double cyc = ms * 1e-3 * clk_khz * 1e3;
  printf("%-22s %.3f warp-inst/clk/SMSP\n", name, warp_inst / (cyc * sms * 4));
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned *o; cudaMalloc(&o, 64);
  printf("SMs %d clock %d kHz\n", sms, clk);
  run<0>("lop3", 1, o, sms, clk);
  run<1>("add-imm", 1, o, sms, clk);
  run<2>("lop3+add-imm", 2, o, sms, clk);
  run<3>("lop3+imad", 2, o, sms, clk);
  run<4>("imad", 1, o, sms, clk);
  run<5>("lop3+isetp+sel", 3, o, sms, clk);
  run<6>("isetp+sel", 2, o, sms, clk);
  run<7>("popc", 1, o, sms, clk);
  run<8>("popc+imad", 2, o, sms, clk);
  run<9>("add-reg", 1, o, sms, clk);
  run<10>("shl-reg", 1, o, sms, clk);
  run<11>("imad.hi", 1, o, sms, clk);
  run<12>("isetp+@p add", 2, o, sms, clk);
  run<13>("lop3+shl", 2, o, sms, clk);
  run<14>("lop3+isetp+sel", 3, o, sms, clk);
  run<15>("lop3+isetp+@p add", 3, o, sms, clk);
  return 0;
}
