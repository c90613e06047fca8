// tcgen05.mma kind::i8 issue-rate microbenchmark (sm_100a): cycles per MMA for
// M=128 (or 64) x N x K=32 u8 MMAs issued back to back by one thread, the A
// operand from shared memory (SS) or from tensor memory (TS), optionally with
// one tcgen05.cp 128x256b per 4 MMAs (the RowSel M=128 pattern) or with four
// other warps writing TMEM (tcgen05.st) meanwhile.  One CTA per SM, every CTA
// runs the same loop; reports the per-CTA average (profiles/r1f_umma.txt).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2604_04696_b200/csrc umma.cu -o umma
#include <cstdio>
#include <cuda_runtime.h>
#include "rowsel_tc.cuh"

using namespace gpir;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}


// ST > 0: warps 1-4 write TMEM (tcgen05.st); ST < 0: warps 1-8 read TMEM (tcgen05.ld, the epilogue pattern);
// ST >= 100: warps 1-8 stream shared memory (ld.shared.v4 + st.shared.v4 of a private 2 KiB block each);
// ST == 60 / 61: one / two warps stream bulk copies (16 KiB, 2-stage rings) into shared memory meanwhile;
// ST == 50 / 51: one / two tcgen05.commit (to mbarriers nobody waits on) after every 16 MMAs
template <int M, int N, bool TA, bool CP, int ST = 0, bool RND = false>
__global__ void __launch_bounds__(288, 1) k_umma(int iters, unsigned long long* out, const uint8_t* src) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, dummy[2];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  // operands: A 4 planes x M x 32 B, B 4 planes x N x 32 B (zeros: data-oblivious)
  for (int i = threadIdx.x; i < (4 * M * 32 + 4 * N * 32) / 16; i += blockDim.x) {
    // RND: random operand bytes (the tensor pipe's rate may depend on the data through power)
    const uint32_t h = RND ? (uint32_t)(i * 2654435761u) ^ (uint32_t)(blockIdx.x * 40503u) : 0u;
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(h, h * 747796405u + 1u, h ^ 0x9E3779B9u, h * 2891336453u + 7u);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&dummy[0], 1);
    mbar_init(&dummy[1], 1);
    mbar_arrive(&dummy[1]);  // phase 0 complete: waits on parity 0 return at once
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (warp == 0) {
    constexpr uint32_t idesc = umma_idesc_u8(M, N);
    const uint32_t sa = smem_u32(sm), sb = sa + 4 * M * 32;
    const uint64_t a0 = umma_desc(sa, M * 16, 128);
    const uint64_t b0 = umma_desc(sb, N * 16, 128);
    const uint32_t ta = tbase + 448;  // 4 x 8 columns of A in TMEM
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int sp = 0; sp < 4; ++sp) {
          if constexpr (TA && CP) tmem_cp_128x256b(ta + 8 * sp, a0 + (uint64_t)(sp * M * 32 >> 4));
#pragma unroll
          for (int tp = 0; tp < 4; ++tp) {
            const int u = sp + tp;
            const uint64_t bd = b0 + (uint64_t)((tp * N * 32) >> 4);
            const uint32_t dcol = tbase + (uint32_t)((u * N) % 448);
            if constexpr (TA)
              umma_i8_ta(dcol, ta + 8 * sp, bd, idesc, 1u);
            else
              umma_i8(dcol, a0 + (uint64_t)(sp * M * 32 >> 4), bd, idesc, 1u);
          }
        }
        if constexpr (ST == 52) {  // the kernel's per-K-step handshake: wait on a completed barrier + fence
          mbar_wait(&dummy[1], 0);
          tc_fence_after();
        }
        if constexpr (ST == 53) tc_fence_after();
        if constexpr (ST == 50 || ST == 51) umma_commit(&dummy[0]);
        if constexpr (ST == 51) umma_commit(&dummy[1]);
      }
      umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
  } else if ((ST == 60 && warp == 1) || (ST == 61 && (warp == 1 || warp == 2))) {
    uint8_t* ring = sm + 4 * M * 32 + 4 * N * 32 + 1024 + (warp - 1) * 32768;
    __shared__ uint64_t tb[2][2];
    uint64_t* fb = tb[warp - 1];
    if ((threadIdx.x & 31) == 0) {
      mbar_init(&fb[0], 1);
      mbar_init(&fb[1], 1);
      fence_mbar_init();
    }
    __syncwarp();
    const int n = iters * 16 * 16 / 600 + 4;  // about one copy per 600 cycles of the MMA loop
    for (int it = 0; it < n; ++it) {
      const int st = it & 1;
      if (it >= 2) mbar_wait(&fb[st], ((it >> 1) - 1) & 1);
      if ((threadIdx.x & 31) == 0) {
        mbar_expect_tx(&fb[st], 16384);
        bulk_g2s(ring + st * 16384, src + ((size_t)(blockIdx.x * 977 + it * 148) % 2048) * 16384, 16384, &fb[st]);
      }
      __syncwarp();
    }
    for (int it = n; it < n + 2; ++it) mbar_wait(&fb[it & 1], ((it >> 1) - 1) & 1);
  } else if (ST >= 100 && warp >= 1 && warp <= 8) {
    uint4* blk = reinterpret_cast<uint4*>(sm + 4 * M * 32 + 4 * N * 32) + (warp - 1) * 128;
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int it = 0; it < iters * (ST - 100); ++it) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        uint4 x = blk[(r * 32 + (threadIdx.x & 31)) & 127];
        acc.x += x.x; acc.y ^= x.y;
        blk[((r + 2) * 32 + (threadIdx.x & 31)) & 127] = acc;
      }
    }
    if (acc.x == 0xFFFFFFFF) out[1] = acc.y;
  } else if (ST < 0 && warp >= 1 && warp <= 8) {
    const uint32_t q = (uint32_t)(warp & 3) * 32;
    uint32_t acc = 0;
    for (int it = 0; it < iters * -ST; ++it) {
      uint32_t v[7][8];
#pragma unroll
      for (int u = 0; u < 7; ++u) tmem_ld8(tbase + (q << 16) + 224 + (warp > 4 ? 16 : 0) + u * 32 % 224, v[u]);
      tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 7; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += v[u][j];
    }
    if (acc == 0xFFFFFFFF) out[1] = acc;
  } else if (ST > 0 && warp >= 1 && warp <= 4) {
    // TMEM writes at full rate into the spare A buffer (columns 480..511) of this warp's lane quadrant,
    // one 4 KiB block (4 x 8 columns) per 16 MMAs' worth: ST = number of x8 stores per MMA-iteration
    const uint32_t q = (uint32_t)(warp & 3) * 32;
    uint32_t v[8];
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 8 + i;
    for (int it = 0; it < iters * ST; ++it) {
#pragma unroll
      for (int sp = 0; sp < 4; ++sp) tmem_st8(tbase + (q << 16) + 480 + 8 * sp, v);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

static const uint8_t* g_src = nullptr;
template <int M, int N, bool TA, bool CP, int ST = 0, bool RND = false>
void run(const char* name, unsigned long long* d, int sms) {
  const int iters = 2000;
  const int smem = 4 * M * 32 + 4 * N * 32 + 1024 + 2 * 32768;
  cudaFuncSetAttribute(k_umma<M, N, TA, CP, ST, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 8);
    k_umma<M, N, TA, CP, ST, RND><<<sms, 288, smem>>>(iters, d, g_src);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", name, cudaGetErrorString(e));
      return;
    }
  }
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / sms / (iters * 16.0);
  printf("%-28s %7.2f cycles/MMA  (floor %d)\n", name, per, (M < 128 ? 128 : M) * N / 256);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  uint8_t* src;
  cudaMalloc(&src, (size_t)32 << 20);
  cudaMemset(src, 0, (size_t)32 << 20);
  g_src = src;
  run<128, 16, false, false>("M128 N16 SS", d, sms);
  run<128, 32, false, false>("M128 N32 SS", d, sms);
  run<128, 64, false, false>("M128 N64 SS", d, sms);
  run<128, 16, true, false>("M128 N16 TS", d, sms);
  run<128, 32, true, false>("M128 N32 TS", d, sms);
  run<128, 64, true, false>("M128 N64 TS", d, sms);
  run<128, 32, true, true>("M128 N32 TS + cp", d, sms);
  run<128, 64, true, true>("M128 N64 TS + cp", d, sms);
  run<128, 32, true, false, 1>("M128 N32 TS + st(1)", d, sms);
  run<128, 32, true, false, 2>("M128 N32 TS + st(2)", d, sms);
  run<128, 64, true, false, 1>("M128 N64 TS + st(1)", d, sms);
  run<128, 32, true, false, -1>("M128 N32 TS + ld(1)", d, sms);
  run<128, 32, true, false, -4>("M128 N32 TS + ld(4)", d, sms);
  run<128, 32, true, true, -1>("M128 N32 TS + cp + ld(1)", d, sms);
  run<64, 64, false, false, -1>("M64 N64 SS + ld(1)", d, sms);
  run<128, 32, true, false, 50>("M128 N32 TS + commit/16", d, sms);
  run<128, 32, true, false, 51>("M128 N32 TS + 2 commits/16", d, sms);
  run<64, 64, false, false, 50>("M64 N64 SS + commit/16", d, sms);
  run<128, 32, true, false, 52>("M128 N32 TS + wait+fence/16", d, sms);
  run<128, 32, true, false, 53>("M128 N32 TS + fence/16", d, sms);
  run<128, 32, true, false, 60>("M128 N32 TS + TMA(1 warp)", d, sms);
  run<128, 32, true, false, 61>("M128 N32 TS + TMA(2 warps)", d, sms);
  run<64, 64, false, false, 61>("M64 N64 SS + TMA(2 warps)", d, sms);
  run<128, 32, true, false, 0, true>("M128 N32 TS random data", d, sms);
  run<128, 32, true, true, 0, true>("M128 N32 TS + cp random", d, sms);
  run<64, 64, false, false, 0, true>("M64 N64 SS random data", d, sms);
  run<128, 32, true, false, 101>("M128 N32 TS + smem(1)", d, sms);
  run<128, 32, true, false, 104>("M128 N32 TS + smem(4)", d, sms);
  run<128, 32, true, true, 101>("M128 N32 TS + cp + smem(1)", d, sms);
  run<64, 64, false, false>("M64 N64 SS", d, sms);
  run<64, 32, false, false>("M64 N32 SS", d, sms);
  return 0;
}
