// RowSel on the 5th-generation tensor cores (tcgen05.mma kind::i8).
//
// out[b, n, comp, p] = sum_k A[m = 2b + comp, k, p] * D[k, n, p] mod q(p)
// (row_select_raw, src/protocol.py:448-492) is 4N independent GEMMs.  Every
// 27-bit residue is split into four byte planes x = sum_s x_s 2^(8s); the
// 16 plane products are u8 x u8 -> s32 GEMMs on the tensor cores,
// accumulated per anti-diagonal u = s + t in TMEM (7 accumulators of
// K * 4 * 255^2 < 2^31 each), and the epilogue recombines
// sum_u C_u 2^(8u) in 64-bit arithmetic (exact: the true dot product is
// < D0 q^2 < 2^64 for D0 <= 1024) and reduces mod q.  Bit-exact with the
// reference's exact integer GEMM.
//
// Operands are pre-packed in HBM in the UMMA canonical K-major no-swizzle
// layout, one contiguous block per (p, 64-byte K chunk) so each pipeline
// stage is two cp.async.bulk copies (UBLKCP):
//   A8[p][c][plane][g][row m][16 B]          (rows = 2B, packed per batch)
//   D8[p][c][ntile][plane][g][row 32][16 B]  (rows = DB columns, packed once)
// Work item = (p, 32-column tile); a persistent CTA per SM runs a multi-stage
// TMA->MMA pipeline (warp 0 producer, warp 1 single-thread MMA issuer,
// warps 2-5 epilogue) with two TMEM accumulator buffers (7 x 32 columns
// each) so the epilogue of one item overlaps the MMAs of the next.
#pragma once
#include "gpir_common.cuh"

namespace gpir {

constexpr int TC_KC = 64;        // K bytes per pipeline stage
constexpr int TC_NT = 32;        // DB columns per work item (MMA N)
constexpr int TC_MAX_STAGES = 8;
constexpr int TC_ACC_COLS = 7 * TC_NT;  // one accumulator buffer
constexpr int TC_THREADS = 192;  // 6 warps

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle (cute SmemDescriptor):
// start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version=1 [46,48), layout 0.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// instruction descriptor: s32 accumulate, u8 x u8, K-major both, N, M=128
__host__ __device__ constexpr uint32_t umma_idesc_u8(int M, int N) {
  return (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------------------
// packing kernels: u32 residues (p innermost) -> byte planes in the canonical
// layout.  One CTA packs 32 p x 4 rows x one 64-byte K chunk (coalesced both
// ways through a 33 KiB smem tile).  Source row r, depth k, slot p lives at
// src[row_off(r) + k * k_stride + p]; rows >= R and k >= Kd are zero.
struct PackSrc {
  const u32* base;
  size_t row_stride_b;   // words between query b's rows (A) / between columns n (D)
  size_t row_stride_c;   // words between the two components (A) / 0 (D)
  int rows_per_b;        // 2 for A (m = 2b + comp), 1 for D
  size_t k_stride;       // words between consecutive k
};

__device__ __forceinline__ size_t pack_src_off(const PackSrc& s, int r) {
  const int b = r / s.rows_per_b, c = r % s.rows_per_b;
  return (size_t)b * s.row_stride_b + (size_t)c * s.row_stride_c;
}

// out block of (p, chunk c, [ntile]): dst + ((p * nchunks + c) * ntiles + nt) * (4 * RT * 64)
// with RT rows per tile (A: RT = R rows, ntiles = 1; D: RT = 32).
__global__ void __launch_bounds__(256)
    k_pack_planes(PackSrc src, int R, int Kd, int KN, int RT, int ntiles, int nchunks, uint8_t* __restrict__ dst) {
  __shared__ u32 tile[4][TC_KC][33];
  const int p0 = blockIdx.x * 32;
  const int r0 = blockIdx.y * 4;
  const int c = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // load: 8 rows x 64 k x 32 p (each warp-instruction reads 128 B of p)
  for (int it = warp; it < 4 * TC_KC; it += 8) {
    const int rr = it / TC_KC, kk = it % TC_KC;
    const int r = r0 + rr, k = c * TC_KC + kk;
    u32 v = 0;
    if (r < R && k < Kd) v = __ldg(src.base + pack_src_off(src, r) + (size_t)k * src.k_stride + p0 + lane);
    tile[rr][kk][lane] = v;
  }
  __syncthreads();
  // store: for each p (32), plane (4), g (4): rows r0..r0+3, 16 B each -> 64 B runs
  for (int it = tid; it < 32 * 4 * 4 * 4; it += 256) {
    const int rr = it & 3, g = (it >> 2) & 3, plane = (it >> 4) & 3, pp = it >> 6;
    const int r = r0 + rr;
    if (r >= R && r >= ((R + RT - 1) / RT) * RT) continue;
    uint32_t w[4];
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t word = 0;
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) {
        const u32 v = tile[rr][g * 16 + q4 * 4 + bb][pp];
        word |= ((v >> (8 * plane)) & 0xFFu) << (8 * bb);
      }
      w[q4] = word;
    }
    const int nt = r / RT, rin = r % RT;
    const size_t blk = (((size_t)(p0 + pp) * nchunks + c) * ntiles + nt) * (size_t)(4 * RT * TC_KC);
    const size_t off = blk + (size_t)plane * RT * TC_KC + ((size_t)g * RT + rin) * 16;
    *reinterpret_cast<uint4*>(dst + off) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  (void)KN;
}

// ---------------------------------------------------------------------------
// the tensor-core GEMM
struct TcArgs {
  const uint8_t* A8;  // [p][c][plane][g][M][16]
  const uint8_t* D8;  // [p][c][nt][plane][g][32][16]
  u32* out;           // (B, d1, 2, KN) standard layout
  int M;              // 2B rows (<= 128)
  int d1, ntiles, nchunks, KN, logn;
  int items;          // KN * ntiles
  int stages;         // pipeline depth (<= TC_MAX_STAGES)
};

__global__ void __launch_bounds__(TC_THREADS, 1) k_rowsel_tc(TcArgs a, Tables tb) {
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t bytesA = 4u * a.M * TC_KC;
  const uint32_t bytesD = 4u * TC_NT * TC_KC;
  const uint32_t stage_bytes = (bytesA + bytesD + 127u) & ~127u;
  uint8_t* stages = tc_smem;
  const int NS = a.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(tc_smem + NS * stage_bytes + 4096);  // +pad: M=128 MMAs over-read
  uint64_t* empty = full + TC_MAX_STAGES;
  uint64_t* tfull = empty + TC_MAX_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // producer
      int s = 0;
      uint32_t ph = 0;
      for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
        const int p = it / a.ntiles, nt = it % a.ntiles;
        for (int c = 0; c < a.nchunks; ++c) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = stages + s * stage_bytes;
          mbar_expect_tx(&full[s], bytesA + bytesD);
          bulk_g2s(sa, a.A8 + ((size_t)p * a.nchunks + c) * bytesA, bytesA, &full[s]);
          bulk_g2s(sa + bytesA, a.D8 + (((size_t)p * a.nchunks + c) * a.ntiles + nt) * bytesD, bytesD, &full[s]);
          if (++s == NS) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = umma_idesc_u8(128, TC_NT);
      int s = 0;
      uint32_t ph = 0;
      int local = 0;
      for (int it = blockIdx.x; it < a.items; it += gridDim.x, ++local) {
        const int ab = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&tempty[ab], aph ^ 1);
        tc_fence_after();
        const uint32_t dcol = tbase + ab * TC_ACC_COLS;
        uint32_t inited = 0;
        for (int c = 0; c < a.nchunks; ++c) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(stages + s * stage_bytes);
          const uint32_t sd = sa + bytesA;
#pragma unroll 1
          for (int ks = 0; ks < TC_KC / 32; ++ks) {
#pragma unroll
            for (int sp = 0; sp < 4; ++sp) {
#pragma unroll
              for (int tp = 0; tp < 4; ++tp) {
                const int u = sp + tp;
                const uint64_t ad = umma_desc(sa + sp * a.M * TC_KC + ks * 2 * a.M * 16, a.M * 16, 128);
                const uint64_t bd = umma_desc(sd + tp * TC_NT * TC_KC + ks * 2 * TC_NT * 16, TC_NT * 16, 128);
                umma_i8(dcol + u * TC_NT, ad, bd, idesc, (inited >> u) & 1);
                inited |= 1u << u;
              }
            }
          }
          umma_commit(&empty[s]);  // smem stage free once these MMAs retire
          if (++s == NS) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit(&tfull[ab]);
      }
    }
  } else {  // epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +31
    const int quad = warp & 3;
    const int m = quad * 32 + lane;
    int local = 0;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x, ++local) {
      const int ab = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      const int p = it / a.ntiles, nt = it % a.ntiles;
      mbar_wait(&tfull[ab], aph);
      tc_fence_after();
      const Modulus M = tb.mod[p >> a.logn];
      const uint32_t tl = tbase + ((uint32_t)(quad * 32) << 16) + ab * TC_ACC_COLS;
#pragma unroll 1
      for (int c8 = 0; c8 < TC_NT; c8 += 8) {
        u64 acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0;
#pragma unroll
        for (int u = 0; u < 7; ++u) {
          uint32_t v[8];
          tmem_ld8(tl + u * TC_NT + c8, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] += (u64)v[j] << (8 * u);
        }
        if (m < a.M) {
          const int b = m >> 1, comp = m & 1;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int n = nt * TC_NT + c8 + j;
            if (n < a.d1) a.out[(((size_t)b * a.d1 + n) * 2 + comp) * a.KN + p] = reduce_u64(acc[j], M);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

}  // namespace gpir
