// cp.async.bulk (TMA bulk copy) global -> shared throughput per SM (sm_100a):
// one CTA per SM streams CHUNK-byte copies from an L2-resident (or HBM-sized)
// source through an NS-stage ring, one elected thread issuing; reports bytes
// per SM-clock and the chip total.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_04696_b200/csrc bulk.cu -o bulk
#include <algorithm>
#include <cstdio>
#include <cuda_runtime.h>
#include "async.cuh"

using namespace gpir;

// par: each stage's chunk is fetched as `par` equal bulk copies (issued by lanes 0..par-1)
__global__ void __launch_bounds__(32, 1) k_bulk(const uint8_t* src, size_t src_bytes, int chunk, int ns, int iters,
                                               int par, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)ns * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const size_t nchunks = src_bytes / chunk;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int s = it % ns;
    if (it >= ns) mbar_wait(&full[s], ((it / ns) - 1) & 1);  // stage's previous copy landed
    const size_t c = ((size_t)blockIdx.x * 7919 + (size_t)it * 148) % nchunks;
    // par > 0: the stage is `par` copies from lanes 0..par-1; par < 0: one copy from lane (it % -par)
    const int issuer = par > 0 ? 0 : it % -par;
    if ((int)threadIdx.x == issuer) mbar_expect_tx(&full[s], chunk);
    __syncwarp();
    if (par > 0 && (int)threadIdx.x < par) {
      const int pc = chunk / par;
      bulk_g2s(sm + (size_t)s * chunk + threadIdx.x * pc, src + c * chunk + threadIdx.x * pc, pc, &full[s]);
    } else if (par < 0 && (int)threadIdx.x == issuer) {
      bulk_g2s(sm + (size_t)s * chunk, src + c * chunk, chunk, &full[s]);
    }
    __syncwarp();
  }
  for (int it = iters; it < iters + ns; ++it) {
    const int s = it % ns;
    mbar_wait(&full[s], ((it / ns) - 1) & 1);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const size_t big = (size_t)4 << 30, small = (size_t)32 << 20;
  uint8_t* src;
  cudaMalloc(&src, big);
  cudaMemset(src, 1, big);
  for (size_t bytes : {small, big}) {
    for (int chunk : {16384, 32768, 65536}) {
      for (int ns : {2, 3, 6}) {
        for (int cps : {1, 2}) {  // CTAs per SM
          if ((size_t)ns * chunk * cps > 200 * 1024) continue;
          const int smem = ns * chunk + 1024;
          cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          const int iters = (int)(((size_t)512 << 20) / chunk / sms / cps);
          for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(d, 0, 8);
            k_bulk<<<sms * cps, 32, smem>>>(src, bytes, chunk, ns, iters, 1, d);
            cudaDeviceSynchronize();
          }
          unsigned long long h;
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          const double cyc = (double)h / (sms * cps);
          const double bpc = (double)iters * chunk / cyc * cps;
          printf("src %5zu MiB chunk %6d stages %d ctas/SM %d: %6.1f B/clk/SM (%6.0f cyc/copy/CTA)\n", bytes >> 20,
                 chunk, ns, cps, bpc, cyc / iters);
        }
      }
    }
  }
  return 0;
}
