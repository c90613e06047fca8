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
// into TMEM once (tcgen05.cp, columns [0, KC)) and feeds the MMAs of every
// 32-column DB tile of that p: A crosses L2 once per unit instead of once per
// column tile (the r1 kernel re-read it d1/32 times, 6.7x the algorithmic
// operand bytes at config 3), and per MMA only the 1 KiB B slice is read from
// shared memory.  The 7 anti-diagonal s32 accumulators (32 columns each, TMEM
// columns [256, 480)) are single-buffered but issued diagonal by diagonal with
// one commit per diagonal: the epilogue drains diagonal u of tile t into u64
// registers while the MMAs of diagonals u+1.. run, and tile t+1 only waits for
// that drain before its own diagonal u.  The next unit's four A planes are
// copied in just before the first diagonal that needs them (tcgen05.cp and
// tcgen05.mma execute in issue order, and plane u was last read by the
// previous tile's diagonal <= u + 3, dozens of MMAs earlier).
//
// One shared-memory ring of 128 * KC-byte slots carries both the A planes
// (128 rows x KC) and the DB tiles (4 planes x 32 columns x KC), each one
// cp.async.bulk: A8[p][mt][plane][KC/16][128][16], D8[p][nt][plane][KC/16][32][16]
// (UMMA canonical K-major, no swizzle).
//
// Output: out_il = 1 writes the ColTor pair layout (the two cts of a ColTor
// pair interleaved word by word, kernels.cuh PAIRS_IL): the thread of row
// m = 2b + comp holds 16 columns = 8 pairs of one p and stores each pair as one
// 8-byte word pair; out_il = 0 writes the standard (B, d1, 2, K*N) layout.
constexpr int TK_NT = 32;
constexpr int TK_ACC0 = 256;  // first accumulator column
constexpr int TK_MAX_SLOTS = 8;

struct TkArgs {
  const uint8_t* A8;
  const uint8_t* D8;
  u32* out;
  int M;       // 2B
  int mtiles;  // 128-row tiles
  int d1, ntiles, KN, logn;
  int KC;      // padded K bytes per plane (multiple of 32, <= 256)
  int units;   // KN * mtiles
  int slots;   // ring depth
  int out_il;
};

__global__ void __launch_bounds__(TC_THREADS, 1) k_rowsel_tk(TkArgs a, Tables tb) {
  extern __shared__ __align__(1024) uint8_t tk_smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t slot_bytes = 128u * (uint32_t)a.KC;
  const int NS = a.slots;
  uint64_t* full = reinterpret_cast<uint64_t*>(tk_smem + (size_t)NS * slot_bytes);
  uint64_t* empty = full + TK_MAX_SLOTS;
  uint64_t* dfull = empty + TK_MAX_SLOTS;
  uint64_t* dempty = dfull + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + 8);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int u = 0; u < 7; ++u) {
      mbar_init(&dfull[u], 1);
      mbar_init(&dempty[u], TC_EPI_WARPS);
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
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int kst = a.KC >> 5;  // MMA K steps (32 bytes each)

  if (warp == 0) {  // producer: per unit the 4 A planes, then the unit's DB tiles
    const uint64_t pol_once = l2_policy_evict_first();
    uint32_t item = 0;
    for (int un = blockIdx.x; un < a.units; un += gridDim.x) {
      const int p = un / a.mtiles, mt = un % a.mtiles;
      for (int it = 0; it < 4 + a.ntiles; ++it, ++item) {
        const uint32_t s = item % NS, ph = (item / NS) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        if (elect_one()) {
          uint8_t* dst = tk_smem + (size_t)s * slot_bytes;
          mbar_expect_tx(&full[s], slot_bytes);
          if (it < 4)
            bulk_g2s_hint(dst, a.A8 + ((size_t)(p * a.mtiles + mt) * 4 + it) * slot_bytes, slot_bytes, &full[s],
                          pol_once);
          else
            bulk_g2s(dst, a.D8 + ((size_t)p * a.ntiles + (it - 4)) * slot_bytes, slot_bytes, &full[s]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {  // MMA issuer: one elected thread runs the whole schedule
    constexpr uint32_t idesc = umma_idesc_u8(128, TK_NT);
    if (elect_one()) {
      uint32_t item = 0, tile = 0;
      const uint32_t acol = (uint32_t)a.KC >> 2;  // TMEM columns per A plane
      for (int un = blockIdx.x; un < a.units; un += gridDim.x) {
        const uint32_t item_a = item;  // the unit's A planes: ring items item_a .. item_a + 3
        item += 4;
        for (int nt = 0; nt < a.ntiles; ++nt, ++item, ++tile) {
          const uint32_t sb = item % NS, phb = (item / NS) & 1;
          const uint32_t bbase = smem_u32(tk_smem + (size_t)sb * slot_bytes);
          const uint32_t tph = (tile & 1) ^ 1;
#pragma unroll 1
          for (int u = 0; u < 7; ++u) {
            if (nt == 0 && u < 4) {  // A plane u of this unit into TMEM columns [u * acol, (u + 1) * acol)
              const uint32_t ia = item_a + u, sa = ia % NS;
              mbar_wait(&full[sa], (ia / NS) & 1);
              tc_fence_after();
              const uint32_t abase = smem_u32(tk_smem + (size_t)sa * slot_bytes);
              for (int ks = 0; ks < kst; ++ks)
                tmem_cp_128x256b(tbase + u * acol + 8 * ks, umma_desc(abase + ks * 4096, 2048, 128));
              umma_commit(&empty[sa]);  // slot free once the copies have landed
            }
            if (u == 0) {
              mbar_wait(&full[sb], phb);
              tc_fence_after();
            }
            mbar_wait(&dempty[u], tph);  // diagonal u of the previous tile drained
            tc_fence_after();
            const uint32_t dcol = tbase + TK_ACC0 + 32 * u;
            const int sp0 = u > 3 ? u - 3 : 0, sp1 = u < 3 ? u : 3;
            for (int sp = sp0; sp <= sp1; ++sp) {
              const int tp = u - sp;
              for (int ks = 0; ks < kst; ++ks)
                umma_i8_ta(dcol, tbase + sp * acol + 8 * ks,
                           umma_desc(bbase + tp * 32 * a.KC + ks * 1024, 512, 128), idesc,
                           (sp == sp0 && ks == 0) ? 0u : 1u);
            }
            umma_commit(&dfull[u]);
          }
          umma_commit(&empty[sb]);  // DB tile free once every diagonal has read it
        }
      }
    }
    __syncwarp();
  } else {  // epilogue warps 2..9: TMEM lanes 32 * (warp % 4) .., columns 16 * half ..
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t lane_base = tbase + ((uint32_t)(quad * 32) << 16) + TK_ACC0 + 16 * half;
    const int P2 = a.d1 >> 1;
    uint32_t tile = 0;
    for (int un = blockIdx.x; un < a.units; un += gridDim.x) {
      const int p = un / a.mtiles, mt = un % a.mtiles;
      const Modulus M = tb.mod[p >> a.logn];
      const int m = mt * 128 + quad * 32 + lane;
      const bool act = m < a.M;
      const int b = m >> 1, comp = m & 1;
      for (int nt = 0; nt < a.ntiles; ++nt, ++tile) {
        u64 acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0;
#pragma unroll
        for (int u = 0; u < 7; ++u) {
          mbar_wait(&dfull[u], tile & 1);
          tc_fence_after();
          uint32_t v[2][8];
          tmem_ld8(lane_base + 32 * u, v[0]);
          tmem_ld8(lane_base + 32 * u + 8, v[1]);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dempty[u]);
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] += (u64)v[j >> 3][j & 7] << (8 * u);
        }
        if (act) {
          const int n0 = nt * TK_NT + 16 * half;
          if (a.out_il) {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              const int pr = (n0 >> 1) + r;
              if (pr < P2) {
                u32* dst = a.out + ((((size_t)b * P2 + pr) * 2 + comp) * a.KN + p) * 2;
                *reinterpret_cast<uint2*>(dst) = make_uint2(reduce_u64(acc[2 * r], M), reduce_u64(acc[2 * r + 1], M));
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int n = n0 + j;
              if (n < a.d1) a.out[(((size_t)b * a.d1 + n) * 2 + comp) * a.KN + p] = reduce_u64(acc[j], M);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

}  // namespace gpir
