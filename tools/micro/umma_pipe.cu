// RowSel M=128 pipeline probe (sm_100a): a bulk-copy producer warp fills an
// NS-stage ring (A 16 KiB + D 4 KiB per stage, L2-resident source) and the MMA
// warp runs the kernel's per-stage pattern -- wait, 4 x tcgen05.cp of the A
// planes into TMEM, 16 MMAs (M128 N32 K32) reading D from the stage, commit the
// stage -- with no epilogue.  Reports cycles per MMA; variants drop the cp
// (A left in TMEM) or the producer (stages pre-filled, no refill).
#include <cstdio>
#include <cuda_runtime.h>
#include "rowsel_tc.cuh"
using namespace gpir;

template <bool CP, bool PROD, bool ONE = false, bool EPI = false>
__global__ void __launch_bounds__(320, 1) k(const uint8_t* src, int iters, int ns, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr uint32_t BA = 16384, BD = 4096, SB = BA + BD;
  __shared__ uint64_t full[12], empty[12];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (EPI && warp >= 2) {  // epilogue-like warps: TMEM loads of 7 diagonals + a shared-memory staging write
    const uint32_t q = (uint32_t)(warp & 3) * 32;
    u32* stg = reinterpret_cast<u32*>(sm + (size_t)ns * SB) + (warp - 2) * 32 * 33;
    uint32_t acc = 0;
    for (int it = 0; it < iters * 2; ++it) {
      uint32_t v[7][8];
#pragma unroll
      for (int u = 0; u < 7; ++u) tmem_ld8(tbase + (q << 16) + u * 32 + 16 * ((warp - 2) >> 2), v[u]);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        u64 x = 0;
#pragma unroll
        for (int u = 0; u < 7; ++u) x += (u64)v[u][j] << (8 * u);
        stg[(threadIdx.x & 31) * 33 + j] = (u32)(x % 134176769u);
      }
      acc += stg[(threadIdx.x & 31) * 33];
    }
    if (acc == 0xFFFFFFFF) out[1] = acc;
  } else if (warp == 1) {  // producer
    int s = 0;
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      if (PROD || it < ns) {
        mbar_wait(&empty[s], ph ^ 1);
        if (elect_one()) {
          const size_t c = ((size_t)blockIdx.x * 977 + (size_t)it * 148) % 1024;
          mbar_expect_tx(&full[s], SB);
          bulk_g2s(sm + s * SB, src + c * SB, BA, &full[s]);
          bulk_g2s(sm + s * SB + BA, src + c * SB + BA, BD, &full[s]);
        }
        __syncwarp();
      }
      if (++s == ns) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (ONE) {  // MMA issuer: one elected thread runs the whole loop (no warp-wide sync per stage)
    constexpr uint32_t idesc = umma_idesc_u8(128, 32);
    if (elect_one()) {
      int s = 0;
      uint32_t ph = 0, ka = 0;
      long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        if (PROD || it < ns) mbar_wait(&full[s], PROD ? ph : 0);
        tc_fence_after();
        const uint32_t sa = smem_u32(sm + s * SB);
        const uint64_t a0 = umma_desc(sa, 128 * 16, 128);
        const uint64_t b0 = umma_desc(sa + BA, 32 * 16, 128);
        const uint32_t ta = tbase + 448 + 32 * (ka & 1);
        if (CP)
          for (int sp = 0; sp < 4; ++sp) tmem_cp_128x256b(ta + 8 * sp, a0 + (uint64_t)(sp * 256));
        const uint32_t dc = tbase + 224 * (it & 1);
#pragma unroll
        for (int sp = 0; sp < 4; ++sp)
#pragma unroll
          for (int tp = 0; tp < 4; ++tp)
            umma_i8_ta(dc + (uint32_t)((sp + tp) * 32), ta + 8 * sp, b0 + (uint64_t)((tp * 32 * 32) >> 4), idesc, 1u);
        if (PROD) umma_commit(&empty[s]);
        ++ka;
        if (++s == ns) {
          s = 0;
          ph ^= 1;
        }
      }
      __shared__ uint64_t fin1;
      mbar_init(&fin1, 1);
      fence_mbar_init();
      umma_commit(&fin1);
      mbar_wait(&fin1, 0);
      long long t1 = clock64();
      atomicAdd(out, (unsigned long long)(t1 - t0));
    }
    __syncwarp();
  } else {  // MMA issuer
    constexpr uint32_t idesc = umma_idesc_u8(128, 32);
    int s = 0;
    uint32_t ph = 0, ka = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (PROD || it < ns) mbar_wait(&full[s], PROD ? ph : 0);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sa = smem_u32(sm + s * SB);
        const uint64_t a0 = umma_desc(sa, 128 * 16, 128);
        const uint64_t b0 = umma_desc(sa + BA, 32 * 16, 128);
        const uint32_t ta = tbase + 448 + 32 * (ka & 1);
        if (CP)
          for (int sp = 0; sp < 4; ++sp) tmem_cp_128x256b(ta + 8 * sp, a0 + (uint64_t)(sp * 256));
#pragma unroll
        for (int sp = 0; sp < 4; ++sp)
#pragma unroll
          for (int tp = 0; tp < 4; ++tp)
            umma_i8_ta(tbase + (uint32_t)(((sp + tp) * 32 + 224 * (it & 1)) % 448), ta + 8 * sp,
                       b0 + (uint64_t)((tp * 32 * 32) >> 4), idesc, 1u);
        if (PROD) umma_commit(&empty[s]);
        ++ka;
      }
      __syncwarp();
      if (++s == ns) {
        s = 0;
        ph ^= 1;
      }
    }
    __shared__ uint64_t fin;
    if (threadIdx.x == 0) {
      mbar_init(&fin, 1);
      fence_mbar_init();
    }
    __syncwarp();
    if (elect_one()) umma_commit(&fin);
    __syncwarp();
    mbar_wait(&fin, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

template <bool CP, bool PROD, bool ONE = false, bool EPI = false>
void run(const char* name, const uint8_t* src, unsigned long long* d, int sms) {
  const int ns = 7, iters = 3000;
  const int smem = ns * 20480 + 2048 + 8 * 32 * 33 * 4;
  cudaFuncSetAttribute(k<CP, PROD, ONE, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 8);
    k<CP, PROD, ONE, EPI><<<sms, EPI ? 320 : 64, smem>>>(src, iters, ns, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", name, cudaGetErrorString(e));
      return;
    }
  }
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %6.2f cycles/MMA\n", name, (double)h / sms / (iters * 16.0));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  uint8_t* src;
  cudaMalloc(&src, (size_t)1024 * 20480);
  cudaMemset(src, 3, (size_t)1024 * 20480);
  run<true, true>("ring + cp + MMA (the kernel)", src, d, sms);
  run<false, true>("ring + MMA (no cp)", src, d, sms);
  run<true, false>("cp + MMA, stages resident", src, d, sms);
  run<false, false>("MMA only, stages resident", src, d, sms);
  run<true, true, true>("1-thread loop: ring + cp + MMA", src, d, sms);
  run<false, true, true>("1-thread loop: ring + MMA", src, d, sms);
  run<true, false, true>("1-thread loop: cp + MMA resident", src, d, sms);
  run<false, false, true>("1-thread loop: MMA only resident", src, d, sms);
  run<true, true, true, true>("1-thread: ring + cp + MMA + epilogue", src, d, sms);
  run<false, false, true, true>("1-thread: MMA only + epilogue", src, d, sms);
  return 0;
}
