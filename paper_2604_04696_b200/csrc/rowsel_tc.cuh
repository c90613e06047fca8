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
//   A8[p][c][mtile][plane][g][row][16 B]     (rows = 2B in tiles of <= 128, per batch)
//   D8[p][c][ntile][plane][g][row 32][16 B]  (rows = DB columns, packed once)
// Work item = (p, NT-column tile, NT = 32 or 64); a persistent CTA per SM runs a multi-stage
// TMA->MMA pipeline (warp 0 producer, warp 1 single-thread MMA issuer,
// warps 2-9 epilogue: two warps per TMEM lane quadrant, each reducing half the
// columns, with the TMEM loads of the next 8 columns in flight).  With NT = 32 there are two TMEM accumulator buffers
// (7 x 32 columns each) so the epilogue of one item overlaps the MMAs of the
// next; NT = 64 halves the A-operand shared-memory reads per MAC instead.
#pragma once
#include "async.cuh"

namespace gpir {

// K bytes per pipeline stage (KC, a kernel template parameter): 64 for the
// M = 64 tiles, 32 (one MMA K step) for M = 128 tiles, whose larger stages
// would otherwise leave room for too few of them next to the epilogue staging
constexpr int TC_MAX_STAGES = 12;
constexpr int TC_EPI_WARPS = 8;  // two warps per TMEM lane quadrant, each owning half the columns
constexpr int TC_THREADS = 64 + 32 * TC_EPI_WARPS;

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
// D += A(tmem) x B(smem): the A operand read from tensor memory (M = 128 lanes, K-major)
__device__ __forceinline__ void umma_i8_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum));
}
// 128 rows x 32 bytes from shared memory (matrix descriptor) into 8 TMEM columns
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t tmem_dst, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem_dst), "l"(sdesc));
}
// commit arriving on the mbarrier at the same offset in every CTA of ctamask
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t ctamask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(ctamask)
               : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.b32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
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
// with RT rows per tile (A: RT = R rows, ntiles = 1; D: RT = 32/64).  One CTA
// covers 128 p x 4 rows x one 16-byte K group: it reads 64 runs of 512 B and
// each thread turns 2 rows x 16 k of one p into 4 planes x 32 contiguous bytes.
constexpr int PK_P = 128, PK_R = 4, PK_K = 16;
__global__ void __launch_bounds__(256)
    k_pack_planes(PackSrc src, int R, int Kd, int RT, int ntiles, int nchunks, int kc, uint8_t* __restrict__ dst) {
  __shared__ __align__(16) u32 tile[PK_R][PK_K][PK_P];
  const int p0 = blockIdx.x * PK_P;
  const int r0 = blockIdx.y * PK_R;
  const int kg = blockIdx.z;  // global 16-byte K group
  const int c = kg / (kc / PK_K), g = kg % (kc / PK_K);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint4 vals[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {  // run index = warp + 8 i: (row, k) pairs, 32 lanes x 16 B = 512 B
    const int run = warp + 8 * i;
    const int rr = run / PK_K, kk = run % PK_K;
    const int r = r0 + rr, k = kg * PK_K + kk;
    vals[i] = make_uint4(0, 0, 0, 0);
    if (r < R && k < Kd)
      vals[i] = __ldg(reinterpret_cast<const uint4*>(src.base + pack_src_off(src, r) + (size_t)k * src.k_stride + p0) +
                      lane);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int run = warp + 8 * i;
    *reinterpret_cast<uint4*>(&tile[run / PK_K][run % PK_K][lane * 4]) = vals[i];  // conflict-free 128-bit
  }
  __syncthreads();
  const int pp = tid & (PK_P - 1);
  const int rp = tid >> 7;  // row pair 0/1
  const int rpad = ((R + RT - 1) / RT) * RT;
  const int r = r0 + 2 * rp;
  if (r >= rpad) return;
  uint32_t w[2][4][4];  // [row][plane][word]
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      u32 v[4];
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) v[bb] = tile[2 * rp + h][q4 * 4 + bb][pp];
#pragma unroll
      for (int pl = 0; pl < 4; ++pl)
        w[h][pl][q4] = __byte_perm(__byte_perm(v[0], v[1], pl | ((pl + 4) << 4)),
                                   __byte_perm(v[2], v[3], pl | ((pl + 4) << 4)), 0x5410);
    }
  const int nt = r / RT, rin = r % RT;  // rows r, r+1 share the tile (RT even)
  const size_t blk = (((size_t)(p0 + pp) * nchunks + c) * ntiles + nt) * (size_t)(4 * RT * kc);
#pragma unroll
  for (int pl = 0; pl < 4; ++pl) {
    uint4* d = reinterpret_cast<uint4*>(dst + blk + (size_t)pl * RT * kc + ((size_t)g * RT + rin) * 16);
    d[0] = make_uint4(w[0][pl][0], w[0][pl][1], w[0][pl][2], w[0][pl][3]);
    d[1] = make_uint4(w[1][pl][0], w[1][pl][1], w[1][pl][2], w[1][pl][3]);
  }
}

// Row-blocked packer: one CTA covers P p x (1024 / P) rows x one 16-byte K
// group, so every warp store is 32 consecutive rows of one (p, plane) -- 512
// contiguous bytes of the canonical layout (k_pack_planes writes 16-byte
// pieces, one per p) -- while the reads are runs of P p (4P bytes).  The shared
// tile is [k][p][row] with a padded p stride RS: conflict-free for the
// row-per-lane reads and for the (row, 4 p) stores of the load phase.
template <int P>
struct Pk2 {
  static constexpr int RR = 1024 / P;                // rows per CTA
  static constexpr int RS = P == 16 ? 66 : 33;       // padded p stride (words)
  static constexpr int SMEM = PK_K * P * RS * 4;
};
template <int P>
__global__ void __launch_bounds__(256)
    k_pack_planes2(PackSrc src, int R, int Kd, int RT, int ntiles, int nchunks, int kc, uint8_t* __restrict__ dst) {
  using C = Pk2<P>;
  extern __shared__ __align__(16) u32 pk2[];  // [k 16][p P][RS]
  const int p0 = blockIdx.x * P;
  const int r0 = blockIdx.y * C::RR;
  const int kg = blockIdx.z;
  const int c = kg / (kc / PK_K), g = kg % (kc / PK_K);
  const int tid = threadIdx.x;
  {  // load: thread -> row r0 + tid / (P / 4), p quarter tid % (P / 4), all 16 k
    const int row = tid / (P / 4), q4 = tid % (P / 4);
    const int r = r0 + row;
    const size_t roff = r < R ? pack_src_off(src, r) : 0;
    uint4 v[PK_K];
#pragma unroll
    for (int k = 0; k < PK_K; ++k) {
      const int kk = kg * PK_K + k;
      v[k] = (r < R && kk < Kd)
                 ? __ldg(reinterpret_cast<const uint4*>(src.base + roff + (size_t)kk * src.k_stride + p0) + q4)
                 : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < PK_K; ++k) {
      u32* t = pk2 + (k * P + 4 * q4) * C::RS + row;
      t[0] = v[k].x;
      t[C::RS] = v[k].y;
      t[2 * C::RS] = v[k].z;
      t[3 * C::RS] = v[k].w;
    }
  }
  __syncthreads();
  const int rpad = ((R + RT - 1) / RT) * RT;
  const int row = tid % C::RR;
  const int r = r0 + row;
  if (r >= rpad) return;
  const int nt = r / RT, rin = r % RT;
#pragma unroll
  for (int i = 0; i < P * C::RR / 256; ++i) {
    const int pp = tid / C::RR + (256 / C::RR) * i;
    u32 w[4][4];  // [plane][word]
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      u32 x[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) x[b] = pk2[((q4 * 4 + b) * P + pp) * C::RS + row];
#pragma unroll
      for (int pl = 0; pl < 4; ++pl)
        w[pl][q4] = __byte_perm(__byte_perm(x[0], x[1], pl | ((pl + 4) << 4)),
                                __byte_perm(x[2], x[3], pl | ((pl + 4) << 4)), 0x5410);
    }
    const size_t blk = (((size_t)(p0 + pp) * nchunks + c) * ntiles + nt) * (size_t)(4 * RT * kc);
#pragma unroll
    for (int pl = 0; pl < 4; ++pl)
      *reinterpret_cast<uint4*>(dst + blk + (size_t)pl * RT * kc + ((size_t)g * RT + rin) * 16) =
          make_uint4(w[pl][0], w[pl][1], w[pl][2], w[pl][3]);
  }
}

// ---------------------------------------------------------------------------
// the tensor-core GEMM
struct TcArgs {
  const uint8_t* A8;  // [p][c][plane][g][M][16]
  const uint8_t* D8;  // [p][c][nt][plane][g][32][16]
  u32* out;           // (B, d1, 2, KN) standard layout
  int M;              // 2B rows (any; tiled by RA)
  int RA, mtiles;     // rows per A tile (<= 128) and A tiles
  int d1, ntiles, nchunks, KN, logn;
  int items;          // KN * ntiles
  int stages;         // pipeline depth (<= TC_MAX_STAGES)
  int nt_outer;       // schedule order inside a block of PST p: (nt, mt) or (mt, nt)
  unsigned long long* prof;  // optional per-CTA cycle counters [grid][8] (GPIR_TC_PROF)
};

// CTA-local work order: blocks of PST consecutive p (round-robin over CTAs),
// each block swept over all (row tile, column tile) pairs, PST items per
// sweep, so the epilogue can stage PST consecutive p in shared memory and
// write full sectors of the p-innermost output.
template <int PST>
struct TcSched {
  int blk, mt, nt, j;
  __device__ __forceinline__ TcSched() : blk(blockIdx.x), mt(0), nt(0), j(0) {}
  __device__ __forceinline__ bool valid(const TcArgs& a) const { return blk * PST < a.KN; }
  __device__ __forceinline__ int p() const { return blk * PST + j; }
  __device__ __forceinline__ void next(const TcArgs& a) {
    if (++j == PST) {
      j = 0;
      if (a.nt_outer) {  // row tiles inner: one DB tile stays hot while every row tile streams past it
        if (++mt == a.mtiles) {
          mt = 0;
          if (++nt == a.ntiles) {
            nt = 0;
            blk += gridDim.x;
          }
        }
      } else if (++nt == a.ntiles) {
        nt = 0;
        if (++mt == a.mtiles) {
          mt = 0;
          blk += gridDim.x;
        }
      }
    }
  }
};

#ifndef TMEM_A_OK
#define TMEM_A_OK 1
#endif

template <int TC_NT, bool M64, int TC_PST, int TC_KC>
__global__ void __launch_bounds__(TC_THREADS, 1) k_rowsel_tc(TcArgs a, Tables tb) {
  using Sched = TcSched<TC_PST>;
  constexpr int TC_ACC_COLS = 7 * TC_NT;
  constexpr int NBUF = (M64 || 2 * TC_ACC_COLS <= 512) ? 2 : 1;
  // A operand from TMEM for M = 128 tiles when two accumulator buffers and two
  // 32-column A slices fit the 512 columns
  constexpr bool TMEM_A = TMEM_A_OK && !M64 && NBUF * TC_ACC_COLS + 64 <= 512;
  static_assert(TC_ACC_COLS <= 512, "accumulators exceed TMEM");
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t bytesA = 4u * a.RA * TC_KC;
  const uint32_t bytesD = 4u * TC_NT * TC_KC;
  const uint32_t stage_bytes = (bytesA + bytesD + 127u) & ~127u;
  uint8_t* stages = tc_smem;
  const int NS = a.stages;
  u32* outbuf = reinterpret_cast<u32*>(tc_smem + NS * stage_bytes + 4096);  // after the MMA over-read pad
  const int OB_ROW = TC_NT + 1;  // padded row: conflict-free column writes
  uint64_t* full = reinterpret_cast<uint64_t*>(outbuf + TC_PST * a.RA * OB_ROW);
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
      mbar_init(&tempty[b], TC_EPI_WARPS);
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

  if (warp == 0) {  // producer: whole warp walks the schedule, one lane issues the bulk copies
    int s = 0;
    uint32_t ph = 0;
    const uint64_t pol_keep = l2_policy_evict_last(), pol_stream = l2_policy_evict_first();
    for (Sched sc; sc.valid(a); sc.next(a)) {
      const int p = sc.p(), nt = sc.nt;
      for (int c = 0; c < a.nchunks; ++c) {
        mbar_wait(&empty[s], ph ^ 1);
        if (elect_one()) {
          uint8_t* sa = stages + s * stage_bytes;
          mbar_expect_tx(&full[s], bytesA + bytesD);
          const uint8_t* ga = a.A8 + (((size_t)p * a.nchunks + c) * a.mtiles + sc.mt) * bytesA;
          const uint8_t* gd = a.D8 + (((size_t)p * a.nchunks + c) * a.ntiles + nt) * bytesD;
          if (a.ntiles > 1) {  // A is re-read once per column tile: keep it in L2, stream D past it
            bulk_g2s_hint(sa, ga, bytesA, &full[s], pol_keep);
            bulk_g2s_hint(sa + bytesA, gd, bytesD, &full[s], pol_stream);
          } else {
            bulk_g2s(sa, ga, bytesA, &full[s]);
            bulk_g2s(sa + bytesA, gd, bytesD, &full[s]);
          }
        }
        __syncwarp();
        if (++s == NS) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: one elected thread runs the whole schedule -- its mbarrier
    // waits, fences and MMAs -- with no warp-wide convergence per stage, which
    // would let the tensor pipe's shallow queue drain (tools/micro/umma_pipe.cu:
    // 43 -> 33 cycles per M128 x N32 MMA with the per-stage tcgen05.cp)
    constexpr uint32_t idesc = umma_idesc_u8(M64 ? 64 : 128, TC_NT);
    if (elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      int local = 0;
      uint32_t ka = 0;                                        // A TMEM double-buffer index (TMEM_A)
      const uint32_t a_ks = (2u * a.RA * 16u) >> 4;         // descriptor step of one 32-byte K step
      const uint32_t a_pl = (uint32_t)(a.RA * TC_KC) >> 4;  // ... of one byte plane
      for (Sched sc; sc.valid(a); sc.next(a), ++local) {
        const int ab = (NBUF == 2) ? (local & 1) : 0;
        const uint32_t aph = (NBUF == 2) ? ((local >> 1) & 1) : (local & 1);
        long long t0 = clock64();
        mbar_wait(&tempty[ab], aph ^ 1);
        long long t1 = clock64();
        if (a.prof) a.prof[blockIdx.x * 8 + 0] += t1 - t0;  // MMA waits for TMEM
        tc_fence_after();
        const uint32_t dcol = M64 ? tbase + ((uint32_t)(16 * ab) << 16) : tbase + ab * TC_ACC_COLS;
        for (int c = 0; c < a.nchunks; ++c) {
          long long t2 = clock64();
          mbar_wait(&full[s], ph);
          long long t3 = clock64();
          if (a.prof) a.prof[blockIdx.x * 8 + 1] += t3 - t2;  // MMA waits for data
          tc_fence_after();
          const uint32_t sa = smem_u32(stages + s * stage_bytes);
          const uint64_t a0 = umma_desc(sa, a.RA * 16, 128);
          const uint64_t b0 = umma_desc(sa + bytesA, TC_NT * 16, 128);
#pragma unroll
          for (int ks = 0; ks < TC_KC / 32; ++ks) {
            // M = 128 tiles: each A plane slice goes to TMEM once (tcgen05.cp) and
            // feeds its four MMAs from there, so per MMA only the B tile is read
            // from shared memory (A: 4 KiB per MMA otherwise: the SMEM-bandwidth bound)
            const uint32_t ta = tbase + (uint32_t)(NBUF * TC_ACC_COLS + 32 * (ka & 1));
            if constexpr (TMEM_A) {
#pragma unroll
              for (int sp = 0; sp < 4; ++sp)
                tmem_cp_128x256b(ta + 8 * sp, a0 + (uint64_t)(sp * a_pl + ks * a_ks));
            }
#pragma unroll
            for (int sp = 0; sp < 4; ++sp) {
#pragma unroll
              for (int tp = 0; tp < 4; ++tp) {
                const int u = sp + tp;
                const bool first = (ks == 0) && (sp == (u > 3 ? u - 3 : 0));  // first product into diagonal u
                const uint64_t bd = b0 + (uint64_t)((tp * TC_NT * TC_KC + ks * 2 * TC_NT * 16) >> 4);
                const uint32_t acc = (c > 0 || !first) ? 1u : 0u;
                if constexpr (TMEM_A) {
                  umma_i8_ta(dcol + u * TC_NT, ta + 8 * sp, bd, idesc, acc);
                } else {
                  const uint64_t ad = a0 + (uint64_t)(sp * a_pl + ks * a_ks);
                  umma_i8(dcol + u * TC_NT, ad, bd, idesc, acc);
                }
              }
            }
            ++ka;
          }
          umma_commit(&empty[s]);  // smem stage free once these MMAs retire
          if (c == a.nchunks - 1) umma_commit(&tfull[ab]);
          if (a.prof) a.prof[blockIdx.x * 8 + 2] += clock64() - t3;  // MMA issue
          if (++s == NS) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else {  // epilogue warps 2..9: TMEM lanes 32*(warp%4) .. +31, column half (warp-2)/4
    constexpr int EPI_T = 32 * TC_EPI_WARPS;
    constexpr int HC = TC_NT / 2;  // columns per epilogue warp
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int etid = (warp - 2) * 32 + lane;
    int local = 0;
    for (Sched sc; sc.valid(a); sc.next(a), ++local) {
      const int ab = (NBUF == 2) ? (local & 1) : 0;
      const uint32_t aph = (NBUF == 2) ? ((local >> 1) & 1) : (local & 1);
      const int p = sc.p(), nt = sc.nt;
      long long e0 = clock64();
      mbar_wait(&tfull[ab], aph);
      long long e1 = clock64();
      if (a.prof && lane == 0 && warp == 2) a.prof[blockIdx.x * 8 + 3] += e1 - e0;  // epilogue waits
      tc_fence_after();
      // tile row held by this thread's TMEM lane for accumulator buffer ab
      const int ml = M64 ? quad * 16 + (lane & 15) : quad * 32 + lane;
      const int m = sc.mt * a.RA + ml;
      const bool mine = M64 ? ((lane >> 4) == ab) : true;
      if ((M64 ? quad * 16 : quad * 32) < a.RA) {
        const Modulus M = tb.mod[p >> a.logn];
        const uint32_t tl = (M64 ? tbase + ((uint32_t)(quad * 32) << 16)
                                 : tbase + ((uint32_t)(quad * 32) << 16) + ab * TC_ACC_COLS) + half * HC;
        u32* orow = outbuf + ((size_t)sc.j * a.RA + ml) * OB_ROW + half * HC;
        const bool act = mine && ml < a.RA && m < a.M;
        // software pipeline: the TMEM loads of group g+1 are in flight while group g is reduced
        uint32_t v[2][7][8];
#pragma unroll
        for (int u = 0; u < 7; ++u) tmem_ld8(tl + u * TC_NT, v[0][u]);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < HC / 8; ++g) {
          const int cb = g & 1;
          if (g + 1 < HC / 8) {
#pragma unroll
            for (int u = 0; u < 7; ++u) tmem_ld8(tl + u * TC_NT + 8 * (g + 1), v[cb ^ 1][u]);
          }
          if (act) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              u64 acc = 0;
#pragma unroll
              for (int u = 0; u < 7; ++u) acc += (u64)v[cb][u][j] << (8 * u);
              orow[8 * g + j] = reduce_u64(acc, M);
            }
          }
          if (g + 1 < HC / 8) tmem_ld_wait();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);  // TMEM buffer free; staging continues
      if (sc.j == TC_PST - 1) {                 // flush TC_PST consecutive p as 16/32-byte runs
        asm volatile("bar.sync 1, %0;" ::"n"(EPI_T) : "memory");
        const int p0 = sc.blk * TC_PST;
        for (int w = etid; w < a.RA * TC_NT; w += EPI_T) {
          const int ml = w / TC_NT, cc = w % TC_NT;
          const int mm = sc.mt * a.RA + ml;
          const int n = nt * TC_NT + cc;
          if (n < a.d1 && mm < a.M) {
            u32 o[TC_PST];
#pragma unroll
            for (int j = 0; j < TC_PST; ++j) o[j] = outbuf[((size_t)j * a.RA + ml) * OB_ROW + cc];
            u32* dw = a.out + (((size_t)(mm >> 1) * a.d1 + n) * 2 + (mm & 1)) * a.KN + p0;
            if constexpr (TC_PST >= 4) {
              uint4* dst = reinterpret_cast<uint4*>(dw);
#pragma unroll
              for (int v = 0; v < TC_PST / 4; ++v) dst[v] = make_uint4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
            } else {
              *reinterpret_cast<uint2*>(dw) = make_uint2(o[0], o[1]);
            }
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(EPI_T) : "memory");
      }
      if (a.prof && lane == 0 && warp == 2) a.prof[blockIdx.x * 8 + 4] += clock64() - e1;  // epilogue work
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

}  // namespace gpir

namespace gpir {


// ---------------------------------------------------------------------------
// RowSel with the A operand resident in tensor memory (k_rowsel_tk): the
// M = 128 row tiles (2B > 64) for d0 <= 256.
//
// Work unit = (p, 128-row tile).  The unit's A operand -- 128 rows x KC bytes x
// 4 byte planes (KC = d0 rounded up to one 32-byte MMA K step) -- is copied
// into TMEM once (tcgen05.cp, columns [0, 4 KC/4)) and feeds the MMAs of every
// 32-column DB tile of that p, so A crosses L2 once per unit and per MMA only
// the 1 KiB B slice is read from shared memory.
//
// Accumulators (TMEM columns [256, 512)): eight 32-column s32 slots, the seven
// anti-diagonals u = s + t of the byte-plane products with the middle one split
// in two (u = 3 has four products), in two groups of four:
//   group A = {u1, u5, u3a, u6} (7 products per K step),
//   group B = {u2, u4, u3b, u0} (9 products per K step).
// Within a group the MMAs of one K step rotate over its four accumulators so
// that consecutive MMAs into one accumulator are >= 3 apart: an MMA that
// accumulates into the previous one's result waits for it (~40 cycles, against
// 16 per M128 x N32 x K32 MMA back to back; measured: 39 cycles per MMA when a
// diagonal's MMAs were issued back to back).  Each group has one commit; the
// epilogue drains group A of tile t while the MMAs of group B run, and the
// MMAs of tile t+1 only wait for the drain of the same group of tile t, so the
// single accumulator set (A takes the other 256 columns) stays busy while the
// epilogue keeps up (one tile = 2048 tensor cycles).
//
// Epilogue: 16 warps, four per TMEM lane quadrant, each reducing 8 columns;
// the diagonals are recombined as lo = C0 + 2^8 C1 + 2^16 C2 + 2^24 C3,
// hi = C4 + 2^8 C5 + 2^16 C6 (64-bit multiply-adds), x = lo + 2^32 hi mod 2^64 --
// exact, since the true dot product is < d0 q^2 < 2^64 -- and reduced mod q.
//
// Output: the P-major tensor Y[p][m][n] (the window's columns innermost; each
// thread stores 32 contiguous bytes), transposed afterwards into the ciphertext
// layout by k_y_to_cts.  The unit owns a single p, so a p-innermost layout
// could only be written 4-8 bytes at a time.
//
// One shared-memory ring of 128 * KC-byte slots carries both the A planes
// (128 rows x KC) and the DB tiles (4 planes x 32 columns x KC), each one
// cp.async.bulk: A8[p][mt][plane][KC/16][128][16], D8[p][nt][plane][KC/16][32][16]
// (UMMA canonical K-major, no swizzle).  nt0 / ntiles_db select a window of DB
// column tiles (the capacity path runs RowSel per column chunk).
constexpr int TK_NT = 32;
constexpr int TK_ACC0 = 256;  // first accumulator column
constexpr int TK_MAX_SLOTS = 8;
constexpr int TK_EPI_WARPS = 16;
constexpr int TK_THREADS = 96 + 32 * TK_EPI_WARPS;  // producer, MMA, 16 epilogue warps, A producer (aring mode)

struct TkArgs {
  const uint8_t* A8;
  const uint8_t* D8;
  u32* out;     // Y[p][M][d1]
  int M;        // 2B
  int mtiles;   // 128-row tiles
  int d1;       // columns of the window
  int ntiles;   // 32-column tiles of the window
  int nt0, ntiles_db;  // first tile of the window, tiles per p in D8
  int KN, logn;
  int KC;       // padded K bytes per plane (multiple of 32, <= 256)
  int units;    // KN * mtiles
  int slots;    // ring depth
  int pair;     // launched as clusters of 2 CTAs (row tiles 2j, 2j + 1 of one p): DB tiles multicast to both
  int aring;    // ring slots 0..3 hold the A planes only (the next unit's A streams in a whole unit ahead), the rest the DB tiles
  unsigned long long* prof;  // optional per-CTA cycle counters [grid][8] (GPIR_TC_PROF)
};

__device__ __forceinline__ void tk_mma(uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
  umma_i8_ta(d, a, b, umma_idesc_u8(128, TK_NT), acc);
}

__global__ void __launch_bounds__(TK_THREADS, 1) k_rowsel_tk(TkArgs a, Tables tb) {
  extern __shared__ __align__(1024) uint8_t tk_smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t slot_bytes = 128u * (uint32_t)a.KC;
  const int NS = a.slots;
  uint64_t* full = reinterpret_cast<uint64_t*>(tk_smem + (size_t)NS * slot_bytes);
  uint64_t* empty = full + TK_MAX_SLOTS;
  uint64_t* dfull = empty + TK_MAX_SLOTS;  // [group]
  uint64_t* dempty = dfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 2);
  // pair mode (a.pair): the cluster's two CTAs take row tiles 2j and 2j + 1 of the
  // same p, so every DB tile is needed by both: CTA r loads the tiles with
  // (tile index % 2 == r) and multicasts them to both; a ring slot is refilled
  // only after both CTAs' MMAs have released it (their commits multicast to
  // both empty barriers: count 2).  Halves the DB bytes each SM pulls from L2
  // and the bulk copies it issues.
  const uint32_t crank = a.pair ? cluster_ctarank() : 0u;
  const int ustart = a.pair ? (int)cluster_id_x() : (int)blockIdx.x;
  const int ustep = a.pair ? (int)cluster_count_x() : (int)gridDim.x;
  const int mtiles_u = a.pair ? a.mtiles / 2 : a.mtiles;  // row-tile units per p
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], a.pair ? 2 : 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&dfull[g], 1);
      mbar_init(&dempty[g], TK_EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (a.pair) cluster_sync_all();  // both CTAs' barriers exist before any multicast reaches them
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int kst = a.KC >> 5;  // MMA K steps (32 bytes each)

  if (a.aring && (warp == 0 || warp == TK_THREADS / 32 - 1)) {
    // dedicated A slots: warp 0 streams the DB tiles through slots 4.., the last warp
    // the A planes through slots 0..3 (plane sp of a unit reuses the slot of plane sp of
    // the previous one, released right after that unit's tcgen05.cp)
    const uint64_t pol_once = l2_policy_evict_first();
    const int NSD = NS - 4;
    uint32_t k = 0, d = 0;
    for (int un = ustart; un < a.units; un += ustep, ++k) {
      const int p = un / mtiles_u, mt = un % mtiles_u;
      if (warp != 0) {
        for (int sp = 0; sp < 4; ++sp) {
          mbar_wait(&empty[sp], (k & 1) ^ 1);
          if (elect_one()) {
            mbar_expect_tx(&full[sp], slot_bytes);
            bulk_g2s_hint(tk_smem + (size_t)sp * slot_bytes, a.A8 + ((size_t)(p * a.mtiles + mt) * 4 + sp) * slot_bytes,
                          slot_bytes, &full[sp], pol_once);
          }
          __syncwarp();
        }
      } else {
        for (int nt = 0; nt < a.ntiles; ++nt, ++d) {
          const uint32_t s = 4 + d % NSD, ph = (d / NSD) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (elect_one()) {
            mbar_expect_tx(&full[s], slot_bytes);
            bulk_g2s(tk_smem + (size_t)s * slot_bytes, a.D8 + ((size_t)p * a.ntiles_db + a.nt0 + nt) * slot_bytes,
                     slot_bytes, &full[s]);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 0) {  // producer: per unit the 4 A planes, then the unit's DB tiles
    const uint64_t pol_once = l2_policy_evict_first();
    uint32_t item = 0;
    for (int un = ustart; un < a.units; un += ustep) {
      const int p = un / mtiles_u, mt = a.pair ? 2 * (un % mtiles_u) + (int)crank : un % mtiles_u;
      // (L2 prefetches of the next unit's A planes and of DB tiles ahead of the ring were
      // measured: no faster, +24% DRAM reads)
      for (int it = 0; it < 4 + a.ntiles; ++it, ++item) {
        const uint32_t s = item % NS, ph = (item / NS) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        if (elect_one()) {
          uint8_t* dst = tk_smem + (size_t)s * slot_bytes;
          mbar_expect_tx(&full[s], slot_bytes);
          if (it < 4)
            bulk_g2s_hint(dst, a.A8 + ((size_t)(p * a.mtiles + mt) * 4 + it) * slot_bytes, slot_bytes, &full[s],
                          pol_once);
          else if (!a.pair)
            bulk_g2s(dst, a.D8 + ((size_t)p * a.ntiles_db + a.nt0 + (it - 4)) * slot_bytes, slot_bytes, &full[s]);
          else if ((uint32_t)((it - 4) & 1) == crank)
            bulk_g2s_mc(dst, a.D8 + ((size_t)p * a.ntiles_db + a.nt0 + (it - 4)) * slot_bytes, slot_bytes, &full[s],
                        (uint16_t)3);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {  // MMA issuer: one elected thread runs the whole schedule
    if (elect_one()) {
      uint32_t item = 0, tile = 0;
      const uint32_t acol = (uint32_t)a.KC >> 2;  // TMEM columns per A plane
      const uint32_t acc0 = tbase + TK_ACC0;
      uint32_t k = 0, d = 0;
      for (int un = ustart; un < a.units; un += ustep, ++k) {
        const uint32_t item_a = item;  // the unit's A planes: ring items item_a .. item_a + 3
        if (!a.aring) item += 4;
        for (int nt = 0; nt < a.ntiles; ++nt, ++item, ++tile, ++d) {
          const uint32_t sb = a.aring ? 4 + d % (NS - 4) : item % NS;
          const uint32_t phb = a.aring ? (d / (NS - 4)) & 1 : (item / NS) & 1;
          const uint64_t b0 = umma_desc(smem_u32(tk_smem + (size_t)sb * slot_bytes), 512, 128);
          const uint32_t bpl = (uint32_t)(32 * a.KC) >> 4;  // descriptor step of one B plane
          const uint32_t tph = (tile & 1) ^ 1;
          long long t0 = clock64();
          if (nt == 0) {  // the unit's four A planes into TMEM columns [sp * acol, (sp + 1) * acol)
            for (int sp = 0; sp < 4; ++sp) {
              const uint32_t ia = item_a + sp, sa = a.aring ? (uint32_t)sp : ia % NS;
              mbar_wait(&full[sa], a.aring ? (k & 1) : (ia / NS) & 1);
              tc_fence_after();
              const uint32_t abase = smem_u32(tk_smem + (size_t)sa * slot_bytes);
              for (int ks = 0; ks < kst; ++ks)
                tmem_cp_128x256b(tbase + sp * acol + 8 * ks, umma_desc(abase + ks * 4096, 2048, 128));
              if (a.pair)  // slot free once the copies have landed (both CTAs count both releases)
                umma_commit_mc(&empty[sa], (uint16_t)3);
              else
                umma_commit(&empty[sa]);
            }
          }
          mbar_wait(&full[sb], phb);
          tc_fence_after();
          long long t1 = clock64();
          mbar_wait(&dempty[0], tph);  // group A of the previous tile drained
          tc_fence_after();
          long long t2 = clock64();
          // group A (7 products per K step): slots 0..3 = u1, u5, u3a, u6
          //   (s, t) = (0,1) (2,3) (0,3) (3,3) (1,0) (3,2) (3,0)
          for (int ks = 0; ks < kst; ++ks) {
            const uint32_t ak = tbase + 8 * ks;
            const uint64_t bk = b0 + (uint64_t)(ks * 64);
            const uint32_t f = ks ? 1u : 0u;
            tk_mma(acc0 + 0, ak + 0 * acol, bk + 1 * bpl, f);
            tk_mma(acc0 + 32, ak + 2 * acol, bk + 3 * bpl, f);
            tk_mma(acc0 + 64, ak + 0 * acol, bk + 3 * bpl, f);
            tk_mma(acc0 + 96, ak + 3 * acol, bk + 3 * bpl, f);
            tk_mma(acc0 + 0, ak + 1 * acol, bk + 0 * bpl, 1u);
            tk_mma(acc0 + 32, ak + 3 * acol, bk + 2 * bpl, 1u);
            tk_mma(acc0 + 64, ak + 3 * acol, bk + 0 * bpl, 1u);
          }
          umma_commit(&dfull[0]);
          mbar_wait(&dempty[1], tph);  // group B of the previous tile drained
          tc_fence_after();
          long long t3 = clock64();
          // group B (9 products per K step): slots 4..7 = u2, u4, u3b, u0
          //   (0,2) (1,3) (1,2) (1,1) (2,2) (0,0) (2,0) (3,1) (2,1)
          for (int ks = 0; ks < kst; ++ks) {
            const uint32_t ak = tbase + 8 * ks;
            const uint64_t bk = b0 + (uint64_t)(ks * 64);
            const uint32_t f = ks ? 1u : 0u;
            tk_mma(acc0 + 128, ak + 0 * acol, bk + 2 * bpl, f);
            tk_mma(acc0 + 160, ak + 1 * acol, bk + 3 * bpl, f);
            tk_mma(acc0 + 192, ak + 1 * acol, bk + 2 * bpl, f);
            tk_mma(acc0 + 128, ak + 1 * acol, bk + 1 * bpl, 1u);
            tk_mma(acc0 + 160, ak + 2 * acol, bk + 2 * bpl, 1u);
            tk_mma(acc0 + 224, ak + 0 * acol, bk + 0 * bpl, f);
            tk_mma(acc0 + 128, ak + 2 * acol, bk + 0 * bpl, 1u);
            tk_mma(acc0 + 160, ak + 3 * acol, bk + 1 * bpl, 1u);
            tk_mma(acc0 + 192, ak + 2 * acol, bk + 1 * bpl, 1u);
          }
          umma_commit(&dfull[1]);
          if (a.pair)  // DB tile free once both groups of both CTAs have read it
            umma_commit_mc(&empty[sb], (uint16_t)3);
          else
            umma_commit(&empty[sb]);
          if (a.prof) {
            long long t4 = clock64();
            a.prof[blockIdx.x * 8 + 1] += t1 - t0;            // waits for data (and the A copies)
            a.prof[blockIdx.x * 8 + (nt == 0 ? 5 : 6)] += t1 - t0;  // ... at unit starts / inside units
            a.prof[blockIdx.x * 8 + 0] += (t2 - t1) + (t3 - t2 - 0);  // waits for drains + group A issue
            a.prof[blockIdx.x * 8 + 2] += t4 - t3;            // group B issue
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < 2 + TK_EPI_WARPS) {  // epilogue warps 2..17: TMEM lanes 32 * (warp % 4) .., columns 8 * cq ..
    const int quad = warp & 3;
    const int cq = (warp - 2) >> 2;
    const uint32_t lb = tbase + ((uint32_t)(quad * 32) << 16) + TK_ACC0 + 8 * cq;
    const bool vec = (a.d1 & 3) == 0;
    uint32_t tile = 0;
    for (int un = ustart; un < a.units; un += ustep) {
      const int p = un / mtiles_u, mt = a.pair ? 2 * (un % mtiles_u) + (int)crank : un % mtiles_u;
      const Modulus M = tb.mod[p >> a.logn];
      const int m = mt * 128 + quad * 32 + lane;
      const bool act = m < a.M;
      u32* yrow = a.out + ((size_t)p * a.M + (act ? m : 0)) * a.d1;
      for (int nt = 0; nt < a.ntiles; ++nt, ++tile) {
        long long e0 = clock64();
        mbar_wait(&dfull[0], tile & 1);
        long long e1 = clock64();
        tc_fence_after();
        uint32_t c1[8], c5[8], c3a[8], c6[8];
        tmem_ld8(lb + 0, c1);
        tmem_ld8(lb + 32, c5);
        tmem_ld8(lb + 64, c3a);
        tmem_ld8(lb + 96, c6);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[0]);
        u64 lo[8], hi[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          lo[j] = (u64)c3a[j] * 16777216u + (u64)c1[j] * 256u;
          hi[j] = (u64)c6[j] * 65536u + (u64)c5[j] * 256u;
        }
        long long e2 = clock64();
        mbar_wait(&dfull[1], tile & 1);
        long long e3 = clock64();
        tc_fence_after();
        uint32_t c2[8], c4[8], c3b[8], c0[8];
        tmem_ld8(lb + 128, c2);
        tmem_ld8(lb + 160, c4);
        tmem_ld8(lb + 192, c3b);
        tmem_ld8(lb + 224, c0);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[1]);
        u32 r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const u64 l = lo[j] + (u64)c2[j] * 65536u + (u64)c3b[j] * 16777216u + c0[j];
          const u64 h = hi[j] + c4[j];
          r[j] = reduce_u64(l + (h << 32), M);
        }
        const int n0 = nt * TK_NT + 8 * cq;
        if (act) {
          if (vec && n0 + 8 <= a.d1) {
            uint4* dst = reinterpret_cast<uint4*>(yrow + n0);
            dst[0] = make_uint4(r[0], r[1], r[2], r[3]);
            dst[1] = make_uint4(r[4], r[5], r[6], r[7]);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (n0 + j < a.d1) yrow[n0 + j] = r[j];
          }
        }
        if (a.prof && lane == 0 && warp == 2) {
          a.prof[blockIdx.x * 8 + 3] += (e1 - e0) + (e3 - e2);     // epilogue waits
          a.prof[blockIdx.x * 8 + 4] += clock64() - e0 - (e1 - e0) - (e3 - e2);  // epilogue work
        }
      }
    }
  }
  __syncthreads();
  if (a.pair) cluster_sync_all();  // no CTA leaves while its peer may still multicast into it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

// Y[p][m][n] (P-major RowSel output of one column window, d1 columns) ->
// the ciphertext layout (b = m >> 1, comp = m & 1):
//   il = 0: standard out[((b * d1s + nb + n) * 2 + comp) * KN + p]   (d1s: columns of the full tensor)
//   il = 1: ColTor pairs interleaved (kernels.cuh PAIRS_IL):
//           out[(((b * d1s / 2 + (nb + n) / 2) * 2 + comp) * KN + p) * 2 + (n & 1)]
// One CTA transposes 64 p x 64 columns of one row m through shared memory:
// 256-byte read runs, 256-byte (il = 0) or 512-byte (il = 1) write runs.
constexpr int YT_P = 64, YT_N = 64;
__global__ void __launch_bounds__(256) k_y_to_cts(const u32* __restrict__ Y, int M, int d1, int KN, u32* __restrict__ out,
                                                  int d1s, int nb, int il) {
  __shared__ u32 t[YT_N][YT_P + 1];
  const int p0 = blockIdx.x * YT_P, m = blockIdx.y, n0 = blockIdx.z * YT_N;
  const int tid = threadIdx.x;
  const bool vec = (d1 & 3) == 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // 64 p rows x 16 chunks of 16 B
    const int w = tid + 256 * i, row = w >> 4, c4 = w & 15;
    const int n = n0 + 4 * c4;
    const u32* src = Y + ((size_t)(p0 + row) * M + m) * d1;
    if (vec && n + 4 <= d1) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + n));
      t[4 * c4][row] = v.x, t[4 * c4 + 1][row] = v.y, t[4 * c4 + 2][row] = v.z, t[4 * c4 + 3][row] = v.w;
    } else {
      for (int j = 0; j < 4; ++j)
        if (n + j < d1) t[4 * c4 + j][row] = __ldg(src + n + j);
    }
  }
  __syncthreads();
  const int b = m >> 1, comp = m & 1;
  if (il) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {  // 32 pairs x 16 chunks of (4 p x 2 elements)
      const int w = tid + 256 * i, pr = w >> 4, pq = w & 15;
      const int n = n0 + 2 * pr;
      if (n + 1 < d1) {
        const int gp = (nb + n) >> 1, e = 2 * pr, pp = 4 * pq;
        uint4* dst =
            reinterpret_cast<uint4*>(out + ((((size_t)b * (d1s >> 1) + gp) * 2 + comp) * KN + p0 + pp) * 2);
        dst[0] = make_uint4(t[e][pp], t[e + 1][pp], t[e][pp + 1], t[e + 1][pp + 1]);
        dst[1] = make_uint4(t[e][pp + 2], t[e + 1][pp + 2], t[e][pp + 3], t[e + 1][pp + 3]);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // 64 columns x 16 chunks of 4 p
      const int w = tid + 256 * i, nl = w >> 4, q4 = w & 15;
      const int n = n0 + nl;
      if (n < d1) {
        const int pp = 4 * q4;
        *reinterpret_cast<uint4*>(out + (((size_t)b * d1s + nb + n) * 2 + comp) * KN + p0 + pp) =
            make_uint4(t[nl][pp], t[nl][pp + 1], t[nl][pp + 2], t[nl][pp + 3]);
      }
    }
  }
}

}  // namespace gpir
