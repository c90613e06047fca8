// bulk-copy pipelining probe (sm_100a): per CTA, `rings` warps each run an
// independent NS-stage ring; a stage is one copy of c1 bytes, plus (c2 > 0) a
// second copy of c2 bytes on the same mbarrier.  Reports bytes/clk per SM and
// cycles per stage per ring.
#include <algorithm>
#include <cstdio>
#include <cuda_runtime.h>
#include "async.cuh"
using namespace gpir;

__global__ void k(const uint8_t* src, size_t src_bytes, int c1, int c2, int ns, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sb = c1 + c2;
  uint8_t* ring = sm + (size_t)w * ns * sb;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)(blockDim.x >> 5) * ns * sb) + w * 16;
  if (lane == 0) {
    for (int s = 0; s < ns; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const size_t nch = src_bytes / sb;
  long long t0 = clock64();
  for (int it = 0; it < iters + ns; ++it) {
    const int s = it % ns;
    if (it >= ns) mbar_wait(&full[s], ((it / ns) - 1) & 1);
    if (it < iters && lane == 0) {
      const size_t c = ((size_t)(blockIdx.x * 8 + w) * 7919 + (size_t)it * 1187) % nch;
      mbar_expect_tx(&full[s], sb);
      bulk_g2s(ring + (size_t)s * sb, src + c * sb, c1, &full[s]);
      if (c2) bulk_g2s(ring + (size_t)s * sb + c1, src + c * sb + c1, c2, &full[s]);
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const size_t bytes = (size_t)32 << 20;
  uint8_t* src;
  cudaMalloc(&src, (size_t)1 << 30);
  cudaMemset(src, 1, (size_t)1 << 30);
  struct Cfg { int c1, c2, ns, rings; };
  for (Cfg g : {Cfg{16384, 0, 6, 1}, Cfg{16384, 4096, 6, 1}, Cfg{20480, 0, 6, 1}, Cfg{16384, 0, 3, 2},
                Cfg{16384, 4096, 3, 2}, Cfg{8192, 0, 6, 2}, Cfg{4096, 0, 8, 4}, Cfg{16384, 0, 2, 4}}) {
    const int smem = g.ns * (g.c1 + g.c2) * g.rings + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = (int)(((size_t)512 << 20) / (g.c1 + g.c2) / sms / g.rings);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(d, 0, 8);
      k<<<sms, 32 * g.rings, smem>>>(src, bytes, g.c1, g.c2, g.ns, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    }
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = (double)h / (sms * g.rings);  // per ring
    printf("c1 %6d c2 %5d stages %d rings %d: %6.1f B/clk/SM  %5.0f cyc/stage/ring\n", g.c1, g.c2, g.ns, g.rings,
           (double)iters * (g.c1 + g.c2) * g.rings / cyc, cyc / iters);
  }
  return 0;
}
