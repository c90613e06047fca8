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
//      lazy forward NTT and a 32-bit Montgomery MAC of digit * key-row for
//      both ciphertext components (key rows fetched at the start of each
//      transform); the epilogue applies the combine of the phase and writes
//      the output limb.
//
// Compared with one CTA per node (which needs 112 KiB of shared memory for
// the digits and exchange buffers, two CTAs per SM) K2 needs only the 32 KiB
// exchange buffer and <= 85 registers, so three CTAs run per SM, and it
// exposes K-fold more CTAs per stage.
#pragma once
#include "kernels.cuh"
#include "rowsel_tc.cuh"

namespace gpir {

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
            if (pairs)
              pair_diff16(src, off + j0, pairs, CT, Mi.q, x);
            else
              ld16(src + off + j0, x);
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
// K2 core: acc{0,1} = sum_{j < NDIG} NTT_i(digit j) * row_j[comp][limb i] * 2^-32
// (mont_mac on lazy transform outputs), row_j = rows(j) (a comp; b comp at
// + K*N).  Shared memory is just the exchange buffer and the accumulators are
// 32-bit, so three CTAs fit per SM; the key rows of digit j are issued at the
// start of its transform and land while the butterflies run.
// Digits come in groups of ELL (one group per input component, `groups` of
// them); the top digit of each group is folded into its key row
// (k_fold_rows), so its term is direct(group, quarter, x) -- the component's
// NTT-domain input -- instead of a transform.
template <int LOGN, int K, int ELL, class RowFn, class DirFn>
__device__ __forceinline__ void k2_mac(NttState& ns, const int* __restrict__ dig, int groups, int i, RowFn&& row,
                                       DirFn&& direct, const Tables& tb, const TwConst& tc, int (&acc0)[16],
                                       int (&acc1)[16]) {
  constexpr int N = 1 << LOGN;
  const int tid = threadIdx.x;
  const Modulus& Mi = tb.mod[i];
  const u32 q = Mi.q, qinv = 0u - Mi.qinv_neg;
  const int i0 = tid << 4;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc0[r] = acc1[r] = 0;
#pragma unroll 1
  for (int g = 0; g < groups; ++g) {
#pragma unroll 1
    for (int j = g * ELL; j < g * ELL + ELL - 1; ++j) {
      const int* dj = dig + (size_t)j * N;
      const u32* ra = row(j) + (size_t)i * N + i0;
      Key16 ka, kb;
      ka.load(ra);
      kb.load(ra + (size_t)K * N);
      ntt_fwd<LOGN, true>(
          ns, tb.fwd + (size_t)i * N, tc.f[i], Mi, [&](int jj) -> u32 { return lift(__ldg(dj + jj), q); },
          [&](int, const u32(&x)[16]) { mont_mac16(x, ka, kb, acc0, acc1, q, qinv); });
    }
    const u32* ra = row(g * ELL + ELL - 1) + (size_t)i * N + i0;
#pragma unroll
    for (int h = 0; h < 4; ++h) {  // in quarters of 4 slots: few live registers
      const uint4 a4 = __ldg(reinterpret_cast<const uint4*>(ra) + h);
      const uint4 b4 = __ldg(reinterpret_cast<const uint4*>(ra + (size_t)K * N) + h);
      u32 x[4];
      direct(g, h, x);
      const u32 av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        mont_mac(acc0[4 * h + rr], x[rr], av[rr], q, qinv);
        mont_mac(acc1[4 * h + rr], x[rr], bv[rr], q, qinv);
      }
    }
  }
}

#ifndef K2_MINB
#define K2_MINB 3
#endif

// K2, ExpandQuery: node (node0 + blockIdx.x / K), output limb blockIdx.x % K.
// The node's input limb i (a and b components, 2 x 16 KiB) is bulk-copied into
// dynamic shared memory at kernel start (one cp.async.bulk pair, mbarrier) and
// lands while the digit transforms run, so the epilogue's automorphism gathers
// (direct term and combine) read shared memory (<= 2-way bank conflicts for
// the stages run here) instead of issuing scattered 4-byte L2 loads.
template <int LOGN>
constexpr size_t k2eq_dyn_smem() {
  return 2 * ((size_t)4 << LOGN) + 16;
}

template <int LOGN, int K, int ELL>
__global__ void __launch_bounds__(NttCfg<LOGN>::T, K2_MINB)
    k_eq_nttmac(const u32* __restrict__ state, int C, int node0, const int* __restrict__ dig, RowsDesc ksk, u32 k_aut,
                const uint2* __restrict__ mono, u32* __restrict__ out, int Cout, Tables tb,
                const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN;
  __shared__ __align__(16) u32 xbuf[NttCfg<LOGN>::XBUF_WORDS];
  NttState ns{xbuf, 0};
  const int tid = threadIdx.x;
  const int ln = blockIdx.x / K, i = blockIdx.x % K;
  const int gn = node0 + ln;
  const int b = gn / C, c = gn % C;
  const size_t CT = 2 * (size_t)K * N;
  const u32* st = state + (size_t)gn * CT;
  extern __shared__ __align__(128) u32 k2_in[];  // [a limb i | b limb i]
  uint64_t* inbar = reinterpret_cast<uint64_t*>(k2_in + 2 * N);
  if (tid == 0) {
    mbar_init(inbar, 1);
    fence_mbar_init();
    mbar_expect_tx(inbar, 2u * N * 4u);
    bulk_g2s(k2_in, st + (size_t)i * N, N * 4u, inbar);
    bulk_g2s(k2_in + N, st + (size_t)(K + i) * N, N * 4u, inbar);
  }
  const u32* in_a = k2_in;
  const u32* in_b = k2_in + N;
  int acc0[16], acc1[16];
  k2_mac<LOGN, K, ELL>(
      ns, dig + (size_t)ln * ELL * N, 1, i, [&](int j) { return ksk.row(b, j, ELL, CT); },
      [&](int, int h, u32(&x)[4]) {
        if (h == 0) mbar_wait(inbar, 0);  // the transforms' barriers order the init before every wait
#pragma unroll
        for (int r = 0; r < 4; ++r) x[r] = in_a[aut_src((tid << 4) + 4 * h + r, k_aut, LOGN)];
      },
      tb, tc, acc0, acc1);
  // combine (src/planner.py:361-363): out[c] = state + s, out[c + C] = X^-2^t (state - s)
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  const int i0 = tid << 4;
  u32* o0 = out + ((size_t)b * Cout + c) * CT;
  u32* o1 = out + ((size_t)b * Cout + c + C) * CT;
  const bool second = c + C < Cout;
#pragma unroll
  for (int h = 0; h < 4; ++h) {  // four quarters of 4 slots: few live registers
    const uint4 ca = reinterpret_cast<const uint4*>(in_a + i0)[h];
    const uint4 cb = reinterpret_cast<const uint4*>(in_b + i0)[h];
    const u32 cav[4] = {ca.x, ca.y, ca.z, ca.w}, cbv[4] = {cb.x, cb.y, cb.z, cb.w};
    u32 xa[4], xb[4], ya[4], yb[4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int r = 4 * h + rr;
      const u32 sa = mont_fin(acc0[r], ELL, M);
      const u32 sb = mod_add(mont_fin(acc1[r], ELL, M), in_b[aut_src(i0 + r, k_aut, LOGN)], q);
      xa[rr] = mod_add(cav[rr], sa, q);
      xb[rr] = mod_add(cbv[rr], sb, q);
      const uint2 w = __ldg(&mono[(size_t)i * N + i0 + r]);
      ya[rr] = csub(mul_shoup(mod_sub(cav[rr], sa, q), w.x, w.y, q), q);
      yb[rr] = csub(mul_shoup(mod_sub(cbv[rr], sb, q), w.x, w.y, q), q);
    }
    reinterpret_cast<uint4*>(o0 + (size_t)i * N + i0)[h] = make_uint4(xa[0], xa[1], xa[2], xa[3]);
    reinterpret_cast<uint4*>(o0 + (size_t)(K + i) * N + i0)[h] = make_uint4(xb[0], xb[1], xb[2], xb[3]);
    if (second) {
      reinterpret_cast<uint4*>(o1 + (size_t)i * N + i0)[h] = make_uint4(ya[0], ya[1], ya[2], ya[3]);
      reinterpret_cast<uint4*>(o1 + (size_t)(K + i) * N + i0)[h] = make_uint4(yb[0], yb[1], yb[2], yb[3]);
    }
  }
}

// K2, external product / ColTor: ct (m0 + blockIdx.x / K), output limb blockIdx.x % K.
// PAIRS (0: plain cts, 1: ColTor pairs, 2: pair-interleaved) is a template
// parameter: with it known the kernel fits 80 registers without spills.
template <int LOGN, int K, int ELL, int PAIRS>
__global__ void __launch_bounds__(NttCfg<LOGN>::T, K2_MINB)
    k_xp_nttmac_t(const u32* __restrict__ in, size_t in_b, int M_per_b, int m0, const int* __restrict__ dig,
                  RowsDesc rows, u32* __restrict__ out, size_t out_b, Tables tb, const __grid_constant__ TwConst tc) {
  constexpr int pairs = PAIRS;
  constexpr int N = 1 << LOGN;
  __shared__ __align__(16) u32 xbuf[NttCfg<LOGN>::XBUF_WORDS];
  NttState ns{xbuf, 0};
  const int tid = threadIdx.x;
  const int lc = blockIdx.x / K, i = blockIdx.x % K;
  const int g = m0 + lc;
  const int b = g / M_per_b, m = g % M_per_b;
  const size_t CT = 2 * (size_t)K * N;
  int acc0[16], acc1[16];
  const u32* src = pairs ? in + (b * in_b + 2 * (size_t)m) * CT : in + (b * in_b + (size_t)m) * CT;
  // digits: a-component's ELL then b-component's ELL, matching rows [0, 2 ELL)
  k2_mac<LOGN, K, ELL>(
      ns, dig + (size_t)lc * 2 * ELL * N, 2, i, [&](int j) { return rows.row(b, j, ELL, CT); },
      [&](int comp, int h, u32(&x)[4]) {
        const size_t off = (size_t)(comp * K + i) * N + (tid << 4) + 4 * h;
        if (pairs) {
          uint4 v, o;
          pair_ld4(src, off, pairs, CT, v, o);
          const u32 q = tb.mod[i].q;
          x[0] = mod_sub(o.x, v.x, q), x[1] = mod_sub(o.y, v.y, q), x[2] = mod_sub(o.z, v.z, q),
          x[3] = mod_sub(o.w, v.w, q);
        } else {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + off));
          x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
        }
      },
      tb, tc, acc0, acc1);
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  const int i0 = tid << 4;
  const u32* ev = in + (b * in_b + 2 * (size_t)m) * CT;  // ColTor: even + (odd - even) ⊡ rgsw (src/planner.py:457-463)
  u32* d = out + (b * out_b + (size_t)m) * CT;
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    u32 sa[4], sb[4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      sa[rr] = mont_fin(acc0[4 * h + rr], 2 * ELL, M);
      sb[rr] = mont_fin(acc1[4 * h + rr], 2 * ELL, M);
    }
    if (pairs) {
      const uint4 ea = pair_even4(ev, (size_t)i * N + i0 + 4 * h, pairs);
      const uint4 eb = pair_even4(ev, (size_t)(K + i) * N + i0 + 4 * h, pairs);
      sa[0] = mod_add(sa[0], ea.x, q); sa[1] = mod_add(sa[1], ea.y, q);
      sa[2] = mod_add(sa[2], ea.z, q); sa[3] = mod_add(sa[3], ea.w, q);
      sb[0] = mod_add(sb[0], eb.x, q); sb[1] = mod_add(sb[1], eb.y, q);
      sb[2] = mod_add(sb[2], eb.z, q); sb[3] = mod_add(sb[3], eb.w, q);
    }
    reinterpret_cast<uint4*>(d + (size_t)i * N + i0)[h] = make_uint4(sa[0], sa[1], sa[2], sa[3]);
    reinterpret_cast<uint4*>(d + (size_t)(K + i) * N + i0)[h] = make_uint4(sb[0], sb[1], sb[2], sb[3]);
  }
}

// runtime `pairs` front end of k_xp_nttmac_t
template <int LOGN, int K, int ELL>
inline cudaError_t launch_xp_nttmac(int grid, cudaStream_t s, const u32* in, size_t in_b, int M_per_b, int m0,
                                    int pairs, const int* dig, RowsDesc rows, u32* out, size_t out_b, const Tables& tb,
                                    const TwConst& tc) {
  constexpr int T = NttCfg<LOGN>::T;
  if (pairs == 0)
    k_xp_nttmac_t<LOGN, K, ELL, 0><<<grid, T, 0, s>>>(in, in_b, M_per_b, m0, dig, rows, out, out_b, tb, tc);
  else if (pairs == 1)
    k_xp_nttmac_t<LOGN, K, ELL, 1><<<grid, T, 0, s>>>(in, in_b, M_per_b, m0, dig, rows, out, out_b, tb, tc);
  else
    k_xp_nttmac_t<LOGN, K, ELL, 2><<<grid, T, 0, s>>>(in, in_b, M_per_b, m0, dig, rows, out, out_b, tb, tc);
  return cudaGetLastError();
}

}  // namespace gpir
