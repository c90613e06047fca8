// Stage-level ("fused") execution of the tree phases, B200 design.
//
// The reference's STAGE_LEVEL executor streams one node at a time through
// iNTT -> Dcp -> per-digit NTT -> MAC (src/planner.py:364-380, 421-434).  On
// B200 a node is split across two kernels so that neither holds more state
// than the SM can keep resident at high occupancy:
//
//   K1 (one CTA per node/ciphertext): automorphism gather (ExpandQuery) or
//      odd - even (ColTor), the inverse NTT of every limb held in registers,
//      then the exact CRT + centered digit extraction in registers; the signed
//      digits (int32, natural coefficient order) go to a per-stage scratch.
//   K2 (one CTA per node x output limb): for every digit, lift mod q_limb,
//      forward NTT and accumulate digit * key-row for both ciphertext
//      components in 64-bit registers; the two key rows of the next digit
//      are prefetched into shared memory with cp.async.bulk on an mbarrier
//      while the current digit is transformed; the epilogue applies the
//      combine of the phase and writes the output limb.
//
// Compared with one CTA per node (which needs 112 KiB of shared memory for
// the digits and exchange buffers) K2 uses 96 KiB with the key double
// buffer, exposes K-fold more CTAs per stage, and never waits on an L2 key
// load inside the MAC.
#pragma once
#include "kernels.cuh"
#include "rowsel_tc.cuh"

namespace gpir {

// K2 shared memory: xbuf (2N words) + keys [2 buffers][2 comps][N words] + 2 mbarriers
template <int LOGN>
constexpr size_t k2_smem_bytes() {
  return (size_t)NttCfg<LOGN>::XBUF_WORDS * 4 + (size_t)4 * (1 << LOGN) * 4 + 2 * 8;
}

// ---------------------------------------------------------------------------
// K1, ExpandQuery: a-component of node (node0 + blockIdx.x), automorphism
// gather, iNTT of all limbs, digits -> dig[(blockIdx.x * ELL + j) * N + coeff]
template <int LOGN, int K, int ELL>
__global__ void __launch_bounds__(NttCfg<LOGN>::T)
    k_eq_dcp(const u32* __restrict__ state, int node0, u32 k_aut, int* __restrict__ dig, Tables tb, CrtConst cc,
             const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN, T = NttCfg<LOGN>::T, SH = NttCfg<LOGN>::SHIFT;
  __shared__ __align__(16) u32 xbuf[NttCfg<LOGN>::XBUF_WORDS];
  NttState ns{xbuf, 0};
  const int tid = threadIdx.x;
  const size_t CT = 2 * (size_t)K * N;
  const u32* st = state + (size_t)(node0 + blockIdx.x) * CT;
  u32 coef[K][16];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    __syncthreads();
    u32* sb = stage_buffer<LOGN>(ns);
    const uint4* src = reinterpret_cast<const uint4*>(st + (size_t)i * N);
    for (int v = tid; v < N / 4; v += T) reinterpret_cast<uint4*>(sb)[v] = __ldg(src + v);
    __syncthreads();
    ntt_inv<LOGN>(
        ns, tb.inv + (size_t)i * N, tc.i[i], tb.mod[i],
        [&](int i0, u32(&x)[16]) {
#pragma unroll
          for (int r = 0; r < 16; ++r) x[r] = sb[aut_src(i0 + r, k_aut, LOGN)];
        },
        [&](int, int r, u32 v) { coef[i][r] = v; });
  }
  int* out = dig + (size_t)blockIdx.x * ELL * N;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    u32 c[K];
#pragma unroll
    for (int i = 0; i < K; ++i) c[i] = coef[i][r];
    int d[ELL];
    dcp_coeff<K, ELL>(c, d, tb, cc);
#pragma unroll
    for (int j = 0; j < ELL; ++j) out[(size_t)j * N + (tid | (r << SH))] = d[j];
  }
}

// K1, external product: ciphertext (m0 + blockIdx.x) of the (B, M) batch (or
// the ColTor pair difference), both components -> 2*ELL digit polynomials
template <int LOGN, int K, int ELL>
__global__ void __launch_bounds__(NttCfg<LOGN>::T)
    k_xp_dcp(const u32* __restrict__ in, size_t in_b, int M_per_b, int m0, int pairs, int* __restrict__ dig,
             Tables tb, CrtConst cc, const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN, SH = NttCfg<LOGN>::SHIFT;
  __shared__ __align__(16) u32 xbuf[NttCfg<LOGN>::XBUF_WORDS];
  NttState ns{xbuf, 0};
  const int tid = threadIdx.x;
  const int g = m0 + blockIdx.x;
  const int b = g / M_per_b, m = g % M_per_b;
  const size_t CT = 2 * (size_t)K * N;
  const u32* src = pairs ? in + (b * in_b + 2 * (size_t)m) * CT : in + (b * in_b + (size_t)m) * CT;
  int* out = dig + (size_t)blockIdx.x * 2 * ELL * N;
#pragma unroll 1
  for (int comp = 0; comp < 2; ++comp) {
    u32 coef[K][16];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const Modulus& Mi = tb.mod[i];
      const size_t off = (size_t)(comp * K + i) * N;
      ntt_inv<LOGN>(
          ns, tb.inv + (size_t)i * N, tc.i[i], Mi,
          [&](int j0, u32(&x)[16]) {
            ld16(src + off + j0, x);
            if (pairs) {
              u32 o[16];
              ld16(src + CT + off + j0, o);
#pragma unroll
              for (int r = 0; r < 16; ++r) x[r] = mod_sub(o[r], x[r], Mi.q);
            }
          },
          [&](int, int r, u32 v) { coef[i][r] = v; });
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      u32 c[K];
#pragma unroll
      for (int i = 0; i < K; ++i) c[i] = coef[i][r];
      int d[ELL];
      dcp_coeff<K, ELL>(c, d, tb, cc);
#pragma unroll
      for (int j = 0; j < ELL; ++j) out[((size_t)comp * ELL + j) * N + (tid | (r << SH))] = d[j];
    }
  }
}

// ---------------------------------------------------------------------------
// K2 core: acc{0,1} = sum_{j < NDIG} NTT_i(digit j) * row_j[comp][limb i],
// row_j = rows(j) (a comp; b comp at + K*N).  Key rows of digit j+1 are
// prefetched into smem while digit j is transformed.
template <int LOGN, int K, class RowFn>
__device__ __forceinline__ void k2_mac(NttState& ns, u32* keys, uint64_t* kbar, const int* __restrict__ dig, int ndig,
                                       int i, RowFn&& row, const Tables& tb, const TwConst& tc, Acc (&acc0)[16],
                                       Acc (&acc1)[16]) {
  constexpr int N = 1 << LOGN, SH = NttCfg<LOGN>::SHIFT;
  const int tid = threadIdx.x;
  const Modulus& Mi = tb.mod[i];
  const u32 q = Mi.q;
  const int i0 = tid << 4;
  auto prefetch = [&](int j) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads before async writes
    const u32* ra = row(j) + (size_t)i * N;
    u32* kb = keys + (size_t)(j & 1) * 2 * N;
    mbar_expect_tx(&kbar[j & 1], 2 * N * 4);
    bulk_g2s(kb, ra, N * 4, &kbar[j & 1]);
    bulk_g2s(kb + N, ra + (size_t)K * N, N * 4, &kbar[j & 1]);
  };
  if (tid == 0) prefetch(0);
#pragma unroll
  for (int r = 0; r < 16; ++r) acc_zero(acc0[r]), acc_zero(acc1[r]);
#pragma unroll 1
  for (int j = 0; j < ndig; ++j) {
    __syncthreads();  // every thread is past the MAC of digit j-1: its key buffer may be refilled
    if (tid == 0 && j + 1 < ndig) prefetch(j + 1);
    const int* dj = dig + (size_t)j * N;
    ntt_fwd<LOGN>(
        ns, tb.fwd + (size_t)i * N, tc.f[i], Mi, [&](int jj) -> u32 { return lift(__ldg(dj + jj), q); },
        [&](int, const u32(&x)[16]) {
          mbar_wait(&kbar[j & 1], (j >> 1) & 1);
          const u32* ka = keys + (size_t)(j & 1) * 2 * N + i0;
          const u32* kb = ka + N;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 a = *reinterpret_cast<const uint4*>(ka + 4 * c);
            const uint4 b = *reinterpret_cast<const uint4*>(kb + 4 * c);
            acc_mac(acc0[4 * c], x[4 * c], a.x);
            acc_mac(acc0[4 * c + 1], x[4 * c + 1], a.y);
            acc_mac(acc0[4 * c + 2], x[4 * c + 2], a.z);
            acc_mac(acc0[4 * c + 3], x[4 * c + 3], a.w);
            acc_mac(acc1[4 * c], x[4 * c], b.x);
            acc_mac(acc1[4 * c + 1], x[4 * c + 1], b.y);
            acc_mac(acc1[4 * c + 2], x[4 * c + 2], b.z);
            acc_mac(acc1[4 * c + 3], x[4 * c + 3], b.w);
          }
        });
  }
  (void)SH;
}

template <int LOGN>
__device__ __forceinline__ void k2_init(u32* smem, NttState& ns, u32*& keys, uint64_t*& kbar) {
  constexpr int N = 1 << LOGN;
  ns.xbuf = smem;
  ns.parity = 0;
  keys = smem + NttCfg<LOGN>::XBUF_WORDS;
  kbar = reinterpret_cast<uint64_t*>(keys + 4 * N);
  if (threadIdx.x == 0) {
    mbar_init(&kbar[0], 1);
    mbar_init(&kbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

// K2, ExpandQuery: node (node0 + blockIdx.x / K), output limb blockIdx.x % K
template <int LOGN, int K, int ELL>
__global__ void __launch_bounds__(NttCfg<LOGN>::T, 2)
    k_eq_nttmac(const u32* __restrict__ state, int C, int node0, const int* __restrict__ dig, RowsDesc ksk, u32 k_aut,
                const uint2* __restrict__ mono, u32* __restrict__ out, int Cout, Tables tb,
                const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN;
  extern __shared__ __align__(128) u32 smem[];
  NttState ns;
  u32* keys;
  uint64_t* kbar;
  k2_init<LOGN>(smem, ns, keys, kbar);
  const int tid = threadIdx.x;
  const int ln = blockIdx.x / K, i = blockIdx.x % K;
  const int gn = node0 + ln;
  const int b = gn / C, c = gn % C;
  const size_t CT = 2 * (size_t)K * N;
  Acc acc0[16], acc1[16];
  k2_mac<LOGN, K>(ns, keys, kbar, dig + (size_t)ln * ELL * N, ELL, i,
                  [&](int j) { return ksk.row(b, j, ELL, CT); }, tb, tc, acc0, acc1);
  // combine (src/planner.py:361-363): out[c] = state + s, out[c + C] = X^-2^t (state - s)
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  const int i0 = tid << 4;
  const u32* st = state + (size_t)gn * CT;
  u32 ca[16], cb[16];
  ld16(st + (size_t)i * N + i0, ca);
  ld16(st + (size_t)(K + i) * N + i0, cb);
  const u32* stb = st + (size_t)(K + i) * N;
  u32 xa[16], xb[16], ya[16], yb[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const u32 sa = reduce_acc(acc0[r], M);
    const u32 sb = mod_add(reduce_acc(acc1[r], M), __ldg(stb + aut_src(i0 + r, k_aut, LOGN)), q);
    xa[r] = mod_add(ca[r], sa, q);
    xb[r] = mod_add(cb[r], sb, q);
    const uint2 w = __ldg(&mono[(size_t)i * N + i0 + r]);
    ya[r] = csub(mul_shoup(mod_sub(ca[r], sa, q), w.x, w.y, q), q);
    yb[r] = csub(mul_shoup(mod_sub(cb[r], sb, q), w.x, w.y, q), q);
  }
  u32* o0 = out + ((size_t)b * Cout + c) * CT;
  st16(o0 + (size_t)i * N + i0, xa);
  st16(o0 + (size_t)(K + i) * N + i0, xb);
  if (c + C < Cout) {
    u32* o1 = out + ((size_t)b * Cout + c + C) * CT;
    st16(o1 + (size_t)i * N + i0, ya);
    st16(o1 + (size_t)(K + i) * N + i0, yb);
  }
}

// K2, external product / ColTor: ct (m0 + blockIdx.x / K), output limb blockIdx.x % K
template <int LOGN, int K, int ELL>
__global__ void __launch_bounds__(NttCfg<LOGN>::T, 2)
    k_xp_nttmac(const u32* __restrict__ in, size_t in_b, int M_per_b, int m0, int pairs, const int* __restrict__ dig,
                RowsDesc rows, u32* __restrict__ out, size_t out_b, Tables tb, const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN;
  extern __shared__ __align__(128) u32 smem[];
  NttState ns;
  u32* keys;
  uint64_t* kbar;
  k2_init<LOGN>(smem, ns, keys, kbar);
  const int tid = threadIdx.x;
  const int lc = blockIdx.x / K, i = blockIdx.x % K;
  const int g = m0 + lc;
  const int b = g / M_per_b, m = g % M_per_b;
  const size_t CT = 2 * (size_t)K * N;
  Acc acc0[16], acc1[16];
  // digits: a-component's ELL then b-component's ELL, matching rows [0, 2 ELL)
  k2_mac<LOGN, K>(ns, keys, kbar, dig + (size_t)lc * 2 * ELL * N, 2 * ELL, i,
                  [&](int j) { return rows.row(b, j, ELL, CT); }, tb, tc, acc0, acc1);
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  const int i0 = tid << 4;
  u32 sa[16], sb[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    sa[r] = reduce_acc(acc0[r], M);
    sb[r] = reduce_acc(acc1[r], M);
  }
  if (pairs) {  // coltor_stage: even + (odd - even) ⊡ rgsw (src/planner.py:457-463)
    const u32* ev = in + (b * in_b + 2 * (size_t)m) * CT;
    u32 ea[16], eb[16];
    ld16(ev + (size_t)i * N + i0, ea);
    ld16(ev + (size_t)(K + i) * N + i0, eb);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      sa[r] = mod_add(sa[r], ea[r], q);
      sb[r] = mod_add(sb[r], eb[r], q);
    }
  }
  u32* d = out + (b * out_b + (size_t)m) * CT;
  st16(d + (size_t)i * N + i0, sa);
  st16(d + (size_t)(K + i) * N + i0, sb);
}

}  // namespace gpir
