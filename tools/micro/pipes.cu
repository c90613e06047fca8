// Integer pipe throughput microbenchmark (sm_100a): warp-instructions per clock per SM
// for IMAD, IMAD.HI, IMAD.WIDE, IADD3, LOP3 with 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
template <int OP>
__global__ void k(unsigned* out, unsigned a, unsigned b) {
  unsigned x[8];
  unsigned long long w[8];
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 7 + i; w[i] = x[i]; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = x[i] * a + b;                       // IMAD
      if (OP == 1) x[i] = __umulhi(x[i], a) + b * 0 ^ x[i];   // IMAD.HI (+LOP)
      if (OP == 2) w[i] = (unsigned long long)(unsigned)w[i] * a + w[i];  // IMAD.WIDE
      if (OP == 3) x[i] = x[i] + a + (x[i] >> 3);             // IADD3 + SHF
      if (OP == 4) x[i] = (x[i] ^ a) & (b | x[i]);            // LOP3
      if (OP == 5) x[i] = __umulhi(x[i], a);                  // pure IMAD.HI chain
    }
  }
  unsigned s = 0;
  for (int i = 0; i < 8; ++i) s += x[i] + (unsigned)w[i] + (unsigned)(w[i] >> 32);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP>
void run(const char* name, unsigned* d) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * 8, block = 256;
  k<OP><<<grid, block>>>(d, 3, 5);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<grid, block>>>(d, 3, 5);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warp_ops = (double)grid * block / 32 * ITERS * 8;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-12s %.3f ms  warp-ops/clk/SM = %.2f\n", name, ms, warp_ops / cycles / sms);
}
int main() {
  unsigned* d; cudaMalloc(&d, 148 * 8 * 256 * 4 * 2);
  run<0>("IMAD", d); run<1>("HI+LOP", d); run<2>("IMAD.WIDE", d); run<3>("IADD3+SHF", d); run<4>("LOP3", d); run<5>("IMAD.HI", d);
  return 0;
}
