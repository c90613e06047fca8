// GPIR server kernels for sm_100a: ExpandQuery (op-level + stage-fused),
// external product (op-level + stage-fused, used by RGSW assembly and
// ColTor), RowSel (CUDA-core, 64-bit lazy accumulation), DB encode and
// layout conversions.  All NTT-domain data is in the brv layout
// (gpir_common.cuh).  Template parameters: LOGN = log2 n, K = RNS limbs,
// ELL = gadget digits.
#pragma once
#include "async.cuh"
#include "ntt.cuh"

namespace gpir {

#ifndef FUSED_MINB
#define FUSED_MINB 2
#endif

// ---------------------------------------------------------------------------
// BFV row addressing: query b's rows [0, ELL) live at lo, rows [ELL, 2 ELL) at
// hi, optionally through a per-query key-slot indirection.
struct RowsDesc {
  const u32* lo;
  size_t lo_b;
  const u32* hi;
  size_t hi_b;
  const int* slot;
  __device__ __forceinline__ const u32* row(int b, int r, int ell, size_t ct) const {
    const size_t s = slot ? (size_t)slot[b] : (size_t)b;
    return r < ell ? lo + s * lo_b + (size_t)r * ct : hi + s * hi_b + (size_t)(r - ell) * ct;
  }
};

__device__ __forceinline__ void ld16(const u32* __restrict__ p, u32 (&x)[16]) {
  const uint4* v = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint4 t = __ldg(v + c);
    x[4 * c] = t.x; x[4 * c + 1] = t.y; x[4 * c + 2] = t.z; x[4 * c + 3] = t.w;
  }
}

__device__ __forceinline__ void st16(u32* p, const u32 (&x)[16]) {
  uint4* v = reinterpret_cast<uint4*>(p);
#pragma unroll
  for (int c = 0; c < 4; ++c) v[c] = make_uint4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
}

// ColTor pair input (coltor_stage, src/planner.py:457-463).  pairs == 1: the even
// ct at src and the odd one at src + CT (the standard layout); pairs == 2: the
// pair interleaved word by word -- element e of the even ct at src[2e], of the
// odd one at src[2e + 1] -- which is what the tensor-core RowSel epilogue
// writes (one 8-byte store per pair and slot, rowsel_tc.cuh k_rowsel_tk).
constexpr int PAIRS_IL = 2;
__device__ __forceinline__ u32 pair_even1(const u32* __restrict__ src, size_t off, int pairs) {
  return pairs == PAIRS_IL ? __ldg(src + 2 * off) : __ldg(src + off);
}
__device__ __forceinline__ u32 pair_diff1(const u32* __restrict__ src, size_t off, int pairs, size_t CT, u32 q) {
  if (pairs == PAIRS_IL) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(src + 2 * off));
    return mod_sub(v.y, v.x, q);
  }
  return mod_sub(__ldg(src + CT + off), __ldg(src + off), q);
}
// 4 consecutive elements of the even and the odd ct (off multiple of 4)
__device__ __forceinline__ void pair_ld4(const u32* __restrict__ src, size_t off, int pairs, size_t CT, uint4& ev,
                                         uint4& od) {
  if (pairs == PAIRS_IL) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(src + 2 * off));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(src + 2 * off) + 1);
    ev = make_uint4(a.x, a.z, b.x, b.z);
    od = make_uint4(a.y, a.w, b.y, b.w);
  } else {
    ev = __ldg(reinterpret_cast<const uint4*>(src + off));
    od = __ldg(reinterpret_cast<const uint4*>(src + CT + off));
  }
}
__device__ __forceinline__ uint4 pair_even4(const u32* __restrict__ src, size_t off, int pairs) {
  if (pairs == PAIRS_IL) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(src + 2 * off));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(src + 2 * off) + 1);
    return make_uint4(a.x, a.z, b.x, b.z);
  }
  return __ldg(reinterpret_cast<const uint4*>(src + off));
}
// odd - even over 16 consecutive elements
__device__ __forceinline__ void pair_diff16(const u32* __restrict__ src, size_t off, int pairs, size_t CT, u32 q,
                                            u32 (&x)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint4 e, o;
    pair_ld4(src, off + 4 * c, pairs, CT, e, o);
    x[4 * c] = mod_sub(o.x, e.x, q), x[4 * c + 1] = mod_sub(o.y, e.y, q);
    x[4 * c + 2] = mod_sub(o.z, e.z, q), x[4 * c + 3] = mod_sub(o.w, e.w, q);
  }
}
__device__ __forceinline__ void pair_even16(const u32* __restrict__ src, size_t off, int pairs, u32 (&x)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 e = pair_even4(src, off + 4 * c, pairs);
    x[4 * c] = e.x, x[4 * c + 1] = e.y, x[4 * c + 2] = e.z, x[4 * c + 3] = e.w;
  }
}

// acc{0,1}[r] += x[r] * row{a,b}[r] over 16 consecutive brv slots, 4 at a time
__device__ __forceinline__ void mac16(const u32 (&x)[16], const u32* __restrict__ ra, const u32* __restrict__ rb,
                                      Acc (&acc0)[16], Acc (&acc1)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(ra) + c);
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(rb) + c);
    acc_mac(acc0[4 * c], x[4 * c], a.x);
    acc_mac(acc0[4 * c + 1], x[4 * c + 1], a.y);
    acc_mac(acc0[4 * c + 2], x[4 * c + 2], a.z);
    acc_mac(acc0[4 * c + 3], x[4 * c + 3], a.w);
    acc_mac(acc1[4 * c], x[4 * c], b.x);
    acc_mac(acc1[4 * c + 1], x[4 * c + 1], b.y);
    acc_mac(acc1[4 * c + 2], x[4 * c + 2], b.z);
    acc_mac(acc1[4 * c + 3], x[4 * c + 3], b.w);
  }
}

// 16 consecutive key words of one row, fetched before the transform that
// consumes them so the L2 latency hides behind the butterflies
struct Key16 {
  uint4 v[4];
  __device__ __forceinline__ void load(const u32* __restrict__ p) {
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = __ldg(reinterpret_cast<const uint4*>(p) + c);
  }
  __device__ __forceinline__ u32 operator[](int r) const {
    const uint4& t = v[r >> 2];
    return (r & 3) == 0 ? t.x : (r & 3) == 1 ? t.y : (r & 3) == 2 ? t.z : t.w;
  }
};

// acc{0,1}[r] += x[r] * k{a,b}[r] * 2^-32 (mont_mac) for lazy NTT outputs x
__device__ __forceinline__ void mont_mac16(const u32 (&x)[16], const Key16& ka, const Key16& kb, int (&acc0)[16],
                                           int (&acc1)[16], u32 q, u32 qinv) {
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    mont_mac(acc0[r], x[r], ka[r], q, qinv);
    mont_mac(acc1[r], x[r], kb[r], q, qinv);
  }
}

// ---------------------------------------------------------------------------
// CRT + centered digits for one coefficient (src/ring.py:456-495,
// src/he.py:346-362): exact 128-bit reconstruction into [0, Q), centering to
// sign/magnitude, then base-2^z_bits digits with the sign-magnitude carry rule.
//
// Fast path (z = 22, 4-word arithmetic on PTX carry chains): S = sum y_i Q/q_i
// < K Q, reduced by the descending multiples of Q; centered; then the
// carry-rule digits in closed form: with T = mag + sum_{j<ell-1} (z/2-1) z^j,
// digit j < ell-1 is bits [jz, jz+z) of T minus (z/2 - 1) and the last digit
// is T >> (ell-1) z (the rule keeps raw == z/2 positive, so the balanced
// digits lie in [-z/2+1, z/2]; pinned against the reference's DigitExtractor
// on crafted boundary coefficients -- raw digit z/2 and z/2+1 at every position,
// carry chains through all ell digits, +-(Q-1)/2 -- by
// tests/test_gpu_parity.py::test_digits_boundary_vectors, vectors from
// tools/make_digit_golden.py).
struct W4 {
  u32 w0, w1, w2, w3;
};

__device__ __forceinline__ W4 w4(u64 lo, u64 hi) { return W4{(u32)lo, (u32)(lo >> 32), (u32)hi, (u32)(hi >> 32)}; }

// S += y * M  (mod 2^128)
__device__ __forceinline__ void w4_mac(W4& S, u32 y, const W4& M) {
  asm("mad.lo.cc.u32 %0, %4, %5, %0;\n\t"
      "madc.lo.cc.u32 %1, %4, %6, %1;\n\t"
      "madc.lo.cc.u32 %2, %4, %7, %2;\n\t"
      "madc.lo.u32 %3, %4, %8, %3;\n\t"
      "mad.hi.cc.u32 %1, %4, %5, %1;\n\t"
      "madc.hi.cc.u32 %2, %4, %6, %2;\n\t"
      "madc.hi.u32 %3, %4, %7, %3;"
      : "+r"(S.w0), "+r"(S.w1), "+r"(S.w2), "+r"(S.w3)
      : "r"(y), "r"(M.w0), "r"(M.w1), "r"(M.w2), "r"(M.w3));
}

// D = A - B; returns the borrow (A < B)
__device__ __forceinline__ bool w4_sub(W4& D, const W4& A, const W4& B) {
  u32 br;
  asm("sub.cc.u32 %0, %5, %9;\n\t"
      "subc.cc.u32 %1, %6, %10;\n\t"
      "subc.cc.u32 %2, %7, %11;\n\t"
      "subc.cc.u32 %3, %8, %12;\n\t"
      "subc.u32 %4, 0, 0;"
      : "=r"(D.w0), "=r"(D.w1), "=r"(D.w2), "=r"(D.w3), "=r"(br)
      : "r"(A.w0), "r"(A.w1), "r"(A.w2), "r"(A.w3), "r"(B.w0), "r"(B.w1), "r"(B.w2), "r"(B.w3));
  return br != 0;
}

__device__ __forceinline__ W4 w4_add(const W4& A, const W4& B) {
  W4 D;
  asm("add.cc.u32 %0, %4, %8;\n\t"
      "addc.cc.u32 %1, %5, %9;\n\t"
      "addc.cc.u32 %2, %6, %10;\n\t"
      "addc.u32 %3, %7, %11;"
      : "=r"(D.w0), "=r"(D.w1), "=r"(D.w2), "=r"(D.w3)
      : "r"(A.w0), "r"(A.w1), "r"(A.w2), "r"(A.w3), "r"(B.w0), "r"(B.w1), "r"(B.w2), "r"(B.w3));
  return D;
}

__device__ __forceinline__ W4 w4_sel(bool p, const W4& A, const W4& B) {
  return W4{p ? A.w0 : B.w0, p ? A.w1 : B.w1, p ? A.w2 : B.w2, p ? A.w3 : B.w3};
}

// bits [s, s + 32) of T, s a compile-time constant
template <int S>
__device__ __forceinline__ u32 w4_bits(const W4& T) {
  constexpr int w = S >> 5, o = S & 31;
  const u32 lo = w == 0 ? T.w0 : w == 1 ? T.w1 : w == 2 ? T.w2 : T.w3;
  const u32 hi = w == 0 ? T.w1 : w == 1 ? T.w2 : w == 2 ? T.w3 : 0u;
  return o == 0 ? lo : __funnelshift_r(lo, hi, o);
}

template <int ZB, int ELL, int J = 0>
__device__ __forceinline__ void w4_digits(const W4& T, u32 sgn, int (&d)[ELL]) {
  if constexpr (J < ELL) {
    int v;
    if constexpr (J < ELL - 1)
      v = (int)(w4_bits<J * ZB>(T) & ((1u << ZB) - 1)) - ((1 << (ZB - 1)) - 1);
    else
      v = (int)w4_bits<J * ZB>(T);
    d[J] = (v ^ (int)sgn) - (int)sgn;  // sgn = 0 or -1
    w4_digits<ZB, ELL, J + 1>(T, sgn, d);
  }
}

template <int K, int ELL>
__device__ __forceinline__ void dcp_coeff(const u32 (&c)[K], int (&d)[ELL], const Tables& tb, const CrtConst& cc) {
  if (cc.z_bits == 22 && ELL * 22 <= 128) {
    W4 S{0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const Modulus& M = tb.mod[i];
      const u32 y = csub(mul_shoup(c[i], M.mhat, M.mhat_sh, M.q), M.q);
      w4_mac(S, y, w4(cc.m_lo[i], cc.m_hi[i]));
    }
    // S < K Q <= P Q (P = next power of two >= K): subtract P/2 Q, ..., 2 Q, Q
    // conditionally (cc.red holds P Q, P/2 Q, ..., Q; the first is never needed)
    constexpr int NR = K <= 1 ? 0 : K <= 2 ? 1 : K <= 4 ? 2 : 3;
#pragma unroll
    for (int t = 1; t <= NR; ++t) {
      W4 D;
      const bool br = w4_sub(D, S, w4(cc.red_lo[t], cc.red_hi[t]));
      S = w4_sel(br, S, D);
    }
    W4 D, mag;
    const bool pos = !w4_sub(D, w4(cc.half_lo, cc.half_hi), S);  // S <= (Q-1)/2
    w4_sub(D, w4(cc.q_lo, cc.q_hi), S);
    mag = w4_sel(pos, S, D);
    const W4 T = w4_add(mag, w4(cc.dc_lo, cc.dc_hi));
    w4_digits<22, ELL>(T, pos ? 0u : ~0u, d);
    return;
  }
  typedef unsigned __int128 u128;
  u128 X = 0;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const Modulus& M = tb.mod[i];
    const u32 y = csub(mul_shoup(c[i], M.mhat, M.mhat_sh, M.q), M.q);
    const u128 m = ((u128)cc.m_hi[i] << 64) | cc.m_lo[i];
    X += m * y;
  }
  for (int t = 0; t < cc.n_red; ++t) {
    const u128 r = ((u128)cc.red_hi[t] << 64) | cc.red_lo[t];
    if (X >= r) X -= r;
  }
  const u128 half = ((u128)cc.half_hi << 64) | cc.half_lo;
  const u128 Q = ((u128)cc.q_hi << 64) | cc.q_lo;
  const bool neg = X > half;
  u128 mag = neg ? Q - X : X;
  const int zb = cc.z_bits;
  const u64 zmask = (1ull << zb) - 1;
  const int zhalf = 1 << (zb - 1);
#pragma unroll
  for (int j = 0; j < ELL; ++j) {
    int v = (int)((u64)mag & zmask);
    mag >>= zb;
    if (j < ELL - 1 && v > zhalf) {
      v -= 1 << zb;
      mag += 1;
    }
    d[j] = neg ? -v : v;
  }
}

__device__ __forceinline__ u32 lift(int d, u32 q) { return d < 0 ? (u32)(d + (int)q) : (u32)d; }

// private (per-thread) smem slot: word index of (slot, r) for this thread
template <int T>
__device__ __forceinline__ int pv(int slot, int r) {
  return (slot * 16 + r) * T + (int)threadIdx.x;
}

// Dcp over the thread's 16 coefficients, in place in private smem:
// coefficient limb i at slot i -> digit j at slot j.
template <int LOGN, int K, int ELL>
__device__ __forceinline__ void dcp_private(int* priv, const Tables& tb, const CrtConst& cc) {
  constexpr int T = NttCfg<LOGN>::T;
#pragma unroll 1
  for (int r = 0; r < 16; ++r) {
    u32 c[K];
#pragma unroll
    for (int i = 0; i < K; ++i) c[i] = (u32)priv[pv<T>(i, r)];
    int d[ELL];
    dcp_coeff<K, ELL>(c, d, tb, cc);
#pragma unroll
    for (int j = 0; j < ELL; ++j) priv[pv<T>(j, r)] = d[j];
  }
}

template <int K, int ELL>
constexpr int priv_slots() {
  return K > ELL ? K : ELL;
}

// ---------------------------------------------------------------------------
// Top-digit fold of gadget key rows.  The gadget digits of a centered
// coefficient satisfy sum_j z^j d_j = a_c exactly, so by linearity of the NTT
//   NTT(d_{l-1}) = z^-(l-1) (A - sum_{j<l-1} z^j NTT(d_j))   (mod q_i)
// with A = NTT(a) the (NTT-domain) input itself.  Hence for any key rows R_j
//   sum_j NTT(d_j) R_j = sum_{j<l-1} NTT(d_j) R'_j + A R'_{l-1},
//   R'_j = R_j - z^(j-(l-1)) R_{l-1},  R'_{l-1} = z^-(l-1) R_{l-1}.
// The server folds every key row group once (evks and RGSW(s) at upload, the
// ColTor RGSW rows when they are assembled) and then transforms only l-1
// digits per component: one forward NTT in every five is replaced by a MAC
// of the input.  Exact modular arithmetic, so bit-identical results.
// One thread per (b, group, word); src may alias dst.
template <int ELL>
__global__ void k_fold_rows(const u32* src, u32* dst, int B, int G, size_t sb, size_t sg, size_t db, size_t dg,
                            int logn, int K, Tables tb, FoldConst fc) {
  const size_t CTW = (size_t)2 * K << logn;
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (size_t)B * G * CTW) return;
  const size_t w = g % CTW, bg = g / CTW;
  const int grp = (int)(bg % G), b = (int)(bg / G);
  const int i = (int)((w >> logn) % K);
  const u32 q = tb.mod[i].q;
  const u32* s = src + b * sb + grp * sg + w;
  u32* d = dst + b * db + grp * dg + w;
  u32 r[ELL];
#pragma unroll
  for (int j = 0; j < ELL; ++j) r[j] = s[(size_t)j * CTW];
  const u32 top = r[ELL - 1];
#pragma unroll
  for (int j = 0; j < ELL - 1; ++j) {
    const uint2 c = fc.w[i][j];
    d[(size_t)j * CTW] = mod_sub(r[j], csub(mul_shoup(top, c.x, c.y, q), q), q);
  }
  const uint2 c = fc.w[i][ELL - 1];
  d[(size_t)(ELL - 1) * CTW] = csub(mul_shoup(top, c.x, c.y, q), q);
}

// ---------------------------------------------------------------------------
// Stage-fused ExpandQuery node (expand_stage STAGE_LEVEL, src/planner.py:364-380):
// one CTA per tree node.  Automorphism gather + iNTT of `a` for all limbs,
// Dcp, then per output limb: ELL digit NTTs, key-switch MAC against the
// client's evk for this stage, and the (c + s, X^-2^t (c - s)) combine.
template <int LOGN, int K, int ELL>
__global__ void __launch_bounds__(NttCfg<LOGN>::T, FUSED_MINB)
    k_eq_fused(const u32* __restrict__ state, int C, u32* __restrict__ out, int Cout, RowsDesc ksk, u32 k_aut,
               const uint2* __restrict__ mono, Tables tb, CrtConst cc, const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN, T = NttCfg<LOGN>::T, SH = NttCfg<LOGN>::SHIFT;
  static_assert(K <= kTwConstLimbs, "const twiddle table holds 4 limbs");
  extern __shared__ __align__(16) u32 smem[];
  NttState ns{smem, 0};
  int* priv = reinterpret_cast<int*>(smem + NttCfg<LOGN>::XBUF_WORDS);
  uint64_t* bar = reinterpret_cast<uint64_t*>(priv + priv_slots<K, ELL>() * 16 * T);
  const int tid = threadIdx.x;
  const int node = blockIdx.x;
  const int b = node / C, c = node % C;
  const size_t CT = 2 * (size_t)K * N;
  const u32* st = state + ((size_t)b * C + c) * CT;

  // all K limbs of `a` land in private slots 0..K-1 with one bulk copy each;
  // the iNTT of limb i gathers (automorphism) from slot i and writes its
  // coefficients back into slot i (a block barrier separates the two)
  static_assert(priv_slots<K, ELL>() >= K, "slot per limb");
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_expect_tx(bar, (uint32_t)(K * N * 4));
#pragma unroll 1
    for (int i = 0; i < K; ++i) bulk_g2s(priv + i * 16 * T, st + (size_t)i * N, N * 4, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);

#pragma unroll 1
  for (int i = 0; i < K; ++i) {
    const u32* slot = reinterpret_cast<const u32*>(priv + i * 16 * T);
    ntt_inv<LOGN>(
        ns, tb.inv + (size_t)i * N, tc.i[i], tb.mod[i],
        [&](int i0, u32(&x)[16]) {
#pragma unroll
          for (int r = 0; r < 16; ++r) x[r] = slot[aut_src(i0 + r, k_aut, LOGN)];
        },
        [&](int, int r, u32 v) { priv[pv<T>(i, r)] = (int)v; });
  }
#ifndef EXP_NO_DCP
  dcp_private<LOGN, K, ELL>(priv, tb, cc);
#endif

  const int i0 = tid << 4;
  const bool second = c + C < Cout;
  u32* o0 = out + ((size_t)b * Cout + c) * CT;
  u32* o1 = out + ((size_t)b * Cout + c + C) * CT;
#pragma unroll 1
  for (int i = 0; i < K; ++i) {
    const Modulus M = tb.mod[i];
    const u32 q = M.q;
    const u32 qinv = 0u - M.qinv_neg;
    const u32* sta = st + (size_t)i * N;
    const u32* stb = st + (size_t)(K + i) * N;
    u32 gb[16];
    int acc0[16], acc1[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) acc0[r] = acc1[r] = 0;
#pragma unroll 1
    for (int j = 0; j < ELL; ++j) {
      const u32* ra = ksk.row(b, j, ELL, CT) + (size_t)i * N;
      Key16 ka, kb;
      ka.load(ra + i0);
      kb.load(ra + (size_t)K * N + i0);
      if (j == ELL - 1) {  // top digit folded into the keys: MAC the automorphed input tau(a) directly
        u32 x[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) x[r] = __ldg(sta + aut_src(i0 + r, k_aut, LOGN));
        mont_mac16(x, ka, kb, acc0, acc1, q, qinv);
        break;
      }
      if (j == ELL - 2) {  // the automorphism gather of b for the combine, in flight during the last transform
#pragma unroll
        for (int r = 0; r < 16; ++r) gb[r] = __ldg(stb + aut_src(i0 + r, k_aut, LOGN));
      }
      ntt_fwd<LOGN, true>(
          ns, tb.fwd + (size_t)i * N, tc.f[i], M, [&](int jj) -> u32 { return lift(priv[pv<T>(j, jj >> SH)], q); },
          [&](int, const u32(&x)[16]) { mont_mac16(x, ka, kb, acc0, acc1, q, qinv); });
    }
    u32 ca[16], cb[16];
    ld16(st + (size_t)i * N + i0, ca);
    ld16(st + (size_t)(K + i) * N + i0, cb);
    u32 xa[16], xb[16], ya[16], yb[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const u32 sa = mont_fin(acc0[r], ELL, M);
      const u32 sb = mod_add(mont_fin(acc1[r], ELL, M), gb[r], q);
      xa[r] = mod_add(ca[r], sa, q);
      xb[r] = mod_add(cb[r], sb, q);
      const uint2 w = __ldg(&mono[(size_t)i * N + i0 + r]);
      ya[r] = csub(mul_shoup(mod_sub(ca[r], sa, q), w.x, w.y, q), q);
      yb[r] = csub(mul_shoup(mod_sub(cb[r], sb, q), w.x, w.y, q), q);
    }
    st16(o0 + (size_t)i * N + i0, xa);
    st16(o0 + (size_t)(K + i) * N + i0, xb);
    if (second) {
      st16(o1 + (size_t)i * N + i0, ya);
      st16(o1 + (size_t)(K + i) * N + i0, yb);
    }
  }
}

// ---------------------------------------------------------------------------
// Stage-fused external product (external_product_batch STAGE_LEVEL,
// src/planner.py:421-434), one CTA per ciphertext.  With `pairs` the input is
// the ColTor pair (even, odd) and the CTA computes even + (odd - even) ⊡ rows
// (coltor_stage, src/planner.py:457-463); otherwise out = in ⊡ rows.
template <int LOGN, int K, int ELL>
__global__ void __launch_bounds__(NttCfg<LOGN>::T, FUSED_MINB)
    k_xp_fused(const u32* __restrict__ in, size_t in_b, int M_per_b, int pairs, u32* __restrict__ out, size_t out_b,
               RowsDesc rows, Tables tb, CrtConst cc, const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN, T = NttCfg<LOGN>::T, SH = NttCfg<LOGN>::SHIFT;
  static_assert(K <= kTwConstLimbs, "const twiddle table holds 4 limbs");
  extern __shared__ __align__(16) u32 smem[];
  NttState ns{smem, 0};
  int* priv = reinterpret_cast<int*>(smem + NttCfg<LOGN>::XBUF_WORDS);
  const int tid = threadIdx.x;
  const int b = blockIdx.x / M_per_b, m = blockIdx.x % M_per_b;
  const size_t CT = 2 * (size_t)K * N;
  const u32* src = pairs ? in + (b * in_b + 2 * (size_t)m) * CT : in + (b * in_b + (size_t)m) * CT;
  u32* dst = out + (b * out_b + (size_t)m) * CT;
  const int i0 = tid << 4;

#pragma unroll 1
  for (int comp = 0; comp < 2; ++comp) {
#pragma unroll 1
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
          [&](int, int r, u32 v) { priv[pv<T>(i, r)] = (int)v; });
    }
#ifndef EXP_NO_DCP
    dcp_private<LOGN, K, ELL>(priv, tb, cc);
#endif
#pragma unroll 1
    for (int i = 0; i < K; ++i) {
      const Modulus Mi = tb.mod[i];
      const u32 q = Mi.q;
      const u32 qinv = 0u - Mi.qinv_neg;
      int acc0[16], acc1[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) acc0[r] = acc1[r] = 0;
#pragma unroll 1
      for (int j = 0; j < ELL; ++j) {
        const u32* ra = rows.row(b, comp * ELL + j, ELL, CT) + (size_t)i * N;
        Key16 ka, kb;
        ka.load(ra + i0);
        kb.load(ra + (size_t)K * N + i0);
        if (j == ELL - 1) {  // folded top digit: MAC this component of the input directly
          const size_t off = (size_t)(comp * K + i) * N + i0;
          u32 x[16];
          if (pairs)
            pair_diff16(src, off, pairs, CT, q, x);
          else
            ld16(src + off, x);
          mont_mac16(x, ka, kb, acc0, acc1, q, qinv);
          break;
        }
        ntt_fwd<LOGN, true>(
            ns, tb.fwd + (size_t)i * N, tc.f[i], Mi, [&](int jj) -> u32 { return lift(priv[pv<T>(j, jj >> SH)], q); },
            [&](int, const u32(&x)[16]) { mont_mac16(x, ka, kb, acc0, acc1, q, qinv); });
      }
      u32 sa[16], sb[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        sa[r] = mont_fin(acc0[r], ELL, Mi);
        sb[r] = mont_fin(acc1[r], ELL, Mi);
      }
      u32* da = dst + (size_t)i * N + i0;
      u32* db = dst + (size_t)(K + i) * N + i0;
      if (comp == 1) {  // add the a-digit half written by this thread in pass 0
        u32 pa[16], pb[16];
        ld16(da, pa);
        ld16(db, pb);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          sa[r] = mod_add(sa[r], pa[r], q);
          sb[r] = mod_add(sb[r], pb[r], q);
        }
        if (pairs) {
          pair_even16(src, (size_t)i * N + i0, pairs, pa);
          pair_even16(src, (size_t)(K + i) * N + i0, pairs, pb);
#pragma unroll
          for (int r = 0; r < 16; ++r) {
            sa[r] = mod_add(sa[r], pa[r], q);
            sb[r] = mod_add(sb[r], pb[r], q);
          }
        }
      }
      st16(da, sa);
      st16(db, sb);
    }
  }
}

// ---------------------------------------------------------------------------
// Operation-level kernels (expand_stage / external_product_batch
// OPERATION_LEVEL, src/planner.py:345-363, 406-420): every primitive runs
// batched over all nodes of a stage and materialises its output.

// (1a) ExpandQuery: automorphism gather + iNTT of `a`; grid (nodes, K).
template <int LOGN, int K>
__global__ void __launch_bounds__(NttCfg<LOGN>::T)
    k_op_eq_intt(const u32* __restrict__ state, int node0, u32 k_aut, u32* __restrict__ coeff, Tables tb,
                 const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN;
  __shared__ __align__(16) u32 xbuf[2 * N];
  NttState ns{xbuf, 0};
  const int nd = blockIdx.x, i = blockIdx.y;
  const u32* row = state + ((size_t)(node0 + nd) * 2 * K + i) * N;
  u32* dst = coeff + ((size_t)nd * K + i) * N;
  // the row arrives by one bulk copy into the exchange buffer the transform
  // does not use; the automorphism gather then reads shared memory
  __shared__ uint64_t bar;
  u32* stage = xbuf + N;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, N * 4u);
    bulk_g2s(stage, row, N * 4u, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  ntt_inv<LOGN>(
      ns, tb.inv + (size_t)i * N, tc.i[i], tb.mod[i],
      [&](int i0, u32(&x)[16]) {
#pragma unroll
#ifndef EQ_INTT_GLOBAL
        for (int r = 0; r < 16; ++r) x[r] = stage[aut_src(i0 + r, k_aut, LOGN)];
#else
        for (int r = 0; r < 16; ++r) x[r] = __ldg(row + aut_src(i0 + r, k_aut, LOGN));
#endif
      },
      [&](int j, int, u32 v) { dst[j] = v; });
}

// (1b) external product: iNTT of both components (or of odd - even); grid (cts*2, K).
template <int LOGN, int K>
__global__ void __launch_bounds__(NttCfg<LOGN>::T)
    k_op_xp_intt(const u32* __restrict__ in, size_t in_b, int M_per_b, int m0, int pairs, u32* __restrict__ coeff,
                 Tables tb, const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN;
  __shared__ __align__(16) u32 xbuf[2 * N];
  NttState ns{xbuf, 0};
  const int poly = blockIdx.x, i = blockIdx.y;
  const int ct = poly >> 1, comp = poly & 1;
  const int g = m0 + ct;
  const int b = g / M_per_b, m = g % M_per_b;
  const size_t CT = 2 * (size_t)K * N;
  const u32* src = pairs ? in + (b * in_b + 2 * (size_t)m) * CT : in + (b * in_b + (size_t)m) * CT;
  const size_t off = (size_t)(comp * K + i) * N;
  const u32 q = tb.mod[i].q;
  u32* dst = coeff + ((size_t)poly * K + i) * N;
  ntt_inv<LOGN>(
      ns, tb.inv + (size_t)i * N, tc.i[i], tb.mod[i],
      [&](int j0, u32(&x)[16]) {
        if (pairs)
          pair_diff16(src, off + j0, pairs, CT, q, x);
        else
          ld16(src + off + j0, x);
      },
      [&](int j, int, u32 v) { dst[j] = v; });
}

// (2) Dcp: one thread per coefficient; coeff [polys][K][N] -> digits [polys][ELL][N].
// Four consecutive coefficients per thread: 128-bit loads and stores keep
// enough bytes in flight to stream at HBM rate.
// ndig < ELL skips the top digits (the pipeline never reads the folded one)
template <int LOGN, int K, int ELL>
__global__ void k_op_dcp(const u32* __restrict__ coeff, int polys, int* __restrict__ digits, Tables tb, CrtConst cc,
                         int ndig) {
  constexpr int N = 1 << LOGN;
  const size_t g = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (g >= (size_t)polys * N) return;
  const size_t p = g >> LOGN, j = g & (N - 1);
  uint4 v[K];
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = __ldg(reinterpret_cast<const uint4*>(coeff + (p * K + i) * N + j));
  int d[4][ELL];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    u32 c[K];
#pragma unroll
    for (int i = 0; i < K; ++i) c[i] = t == 0 ? v[i].x : t == 1 ? v[i].y : t == 2 ? v[i].z : v[i].w;
    dcp_coeff<K, ELL>(c, d[t], tb, cc);
  }
#pragma unroll
  for (int e = 0; e < ELL; ++e)
    if (e < ndig)
      *reinterpret_cast<int4*>(digits + (p * ELL + e) * N + j) = make_int4(d[0][e], d[1][e], d[2][e], d[3][e]);
}

// (3) digit NTT: grid (polys*(ELL-1), K): lift digit mod q_i, forward NTT
// (the top digit is folded into the keys, k_fold_rows).
template <int LOGN, int K, int ELL>
__global__ void __launch_bounds__(NttCfg<LOGN>::T)
    k_op_digit_ntt(const int* __restrict__ digits, u32* __restrict__ dn, Tables tb, const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN;
  __shared__ __align__(16) u32 xbuf[2 * N];
  NttState ns{xbuf, 0};
  const int pe = (blockIdx.x / (ELL - 1)) * ELL + blockIdx.x % (ELL - 1), i = blockIdx.y;
  const int* src = digits + (size_t)pe * N;
  const u32 q = tb.mod[i].q;
  u32* dst = dn + ((size_t)pe * K + i) * N;
#ifndef DNTT_STAGE
#define DNTT_STAGE 1
#endif
#if DNTT_STAGE
  // the digit row arrives by one bulk copy into the exchange buffer the transform does not use
  __shared__ uint64_t bar;
  const int* stage = reinterpret_cast<const int*>(xbuf + N);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, N * 4u);
    bulk_g2s(xbuf + N, src, N * 4u, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
#else
  const int* stage = src;
#endif
  // lazy outputs (< (2 log n + 1) q < 2^32): the 64-bit MACs take them as they are
  // (ELL terms of < 25 q * q per accumulator, < 2^62)
  ntt_fwd<LOGN, true>(
      ns, tb.fwd + (size_t)i * N, tc.f[i], tb.mod[i], [&](int j) -> u32 { return lift(stage[j], q); },
      [&](int i0, const u32(&x)[16]) { st16(dst + i0, x); });
}

// (4a) ExpandQuery key-switch MAC + combine; one thread per (node, limb, slot).
template <int LOGN, int K, int ELL>
__global__ void k_op_eq_mac(const u32* __restrict__ state, int C, int node0, int nodes, const u32* __restrict__ dn,
                            RowsDesc ksk, u32 k_aut, const uint2* __restrict__ mono, u32* __restrict__ out, int Cout,
                            Tables tb) {
  constexpr int N = 1 << LOGN;
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (size_t)nodes * K * N) return;
  const int pos = (int)(g & (N - 1));
  const int i = (int)((g >> LOGN) % K);
  const int nd = (int)(g / ((size_t)K * N));
  const int gn = node0 + nd;
  const int b = gn / C, c = gn % C;
  const size_t CT = 2 * (size_t)K * N;
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  const u32* st = state + (size_t)gn * CT;
  u64 a0 = 0, a1 = 0;
#pragma unroll
  for (int j = 0; j < ELL; ++j) {  // digit ELL-1 is folded: its term is tau(a) itself
    const u32 d = j < ELL - 1 ? __ldg(dn + (((size_t)nd * ELL + j) * K + i) * N + pos)
                              : __ldg(st + (size_t)i * N + aut_src(pos, k_aut, LOGN));
    const u32* ra = ksk.row(b, j, ELL, CT) + (size_t)i * N + pos;
    a0 += (u64)d * __ldg(ra);
    a1 += (u64)d * __ldg(ra + (size_t)K * N);
  }
  const u32 ca = __ldg(st + (size_t)i * N + pos), cb = __ldg(st + (size_t)(K + i) * N + pos);
  const u32 sa = reduce_u64(a0, M);
  const u32 sb = mod_add(reduce_u64(a1, M), __ldg(st + (size_t)(K + i) * N + aut_src(pos, k_aut, LOGN)), q);
  u32* o0 = out + ((size_t)b * Cout + c) * CT;
  o0[(size_t)i * N + pos] = mod_add(ca, sa, q);
  o0[(size_t)(K + i) * N + pos] = mod_add(cb, sb, q);
  if (c + C < Cout) {
    u32* o1 = out + ((size_t)b * Cout + c + C) * CT;
    const uint2 w = __ldg(&mono[(size_t)i * N + pos]);
    o1[(size_t)i * N + pos] = csub(mul_shoup(mod_sub(ca, sa, q), w.x, w.y, q), q);
    o1[(size_t)(K + i) * N + pos] = csub(mul_shoup(mod_sub(cb, sb, q), w.x, w.y, q), q);
  }
}

// (4a') the same with NB consecutive nodes per thread: the nodes of one query at
// one stage share their key rows, so each thread loads the 2 ELL key values of
// its (limb, slot) once for NB nodes (reloading only where the group crosses
// into the next query) -- the key rows are most of the MAC's memory traffic.
template <int LOGN, int K, int ELL, int NB>
__global__ void k_op_eq_mac_nb(const u32* __restrict__ state, int C, int node0, int nodes, const u32* __restrict__ dn,
                               RowsDesc ksk, u32 k_aut, const uint2* __restrict__ mono, u32* __restrict__ out,
                               int Cout, Tables tb) {
  constexpr int N = 1 << LOGN;
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t groups = ((size_t)nodes + NB - 1) / NB;
  if (g >= groups * K * N) return;
  const int pos = (int)(g & (N - 1));
  const int i = (int)((g >> LOGN) % K);
  const int nd0 = (int)(g / ((size_t)K * N)) * NB;
  const size_t CT = 2 * (size_t)K * N;
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  const u32 src_pos = aut_src(pos, k_aut, LOGN);
  const uint2 w = __ldg(&mono[(size_t)i * N + pos]);
  int cur_b = -1;
  u32 ka[ELL], kb[ELL];
#pragma unroll 1
  for (int u = 0; u < NB; ++u) {
    const int nd = nd0 + u;
    if (nd >= nodes) break;
    const int gn = node0 + nd;
    const int b = gn / C, c = gn % C;
    if (b != cur_b) {
#pragma unroll
      for (int j = 0; j < ELL; ++j) {
        const u32* ra = ksk.row(b, j, ELL, CT) + (size_t)i * N + pos;
        ka[j] = __ldg(ra);
        kb[j] = __ldg(ra + (size_t)K * N);
      }
      cur_b = b;
    }
    const u32* st = state + (size_t)gn * CT;
    u64 a0 = 0, a1 = 0;
#pragma unroll
    for (int j = 0; j < ELL; ++j) {  // digit ELL-1 is folded: its term is tau(a) itself
      const u32 d = j < ELL - 1 ? __ldg(dn + (((size_t)nd * ELL + j) * K + i) * N + pos) : __ldg(st + (size_t)i * N + src_pos);
      a0 += (u64)d * ka[j];
      a1 += (u64)d * kb[j];
    }
    const u32 ca = __ldg(st + (size_t)i * N + pos), cb = __ldg(st + (size_t)(K + i) * N + pos);
    const u32 sa = reduce_u64(a0, M);
    const u32 sb = mod_add(reduce_u64(a1, M), __ldg(st + (size_t)(K + i) * N + src_pos), q);
    u32* o0 = out + ((size_t)b * Cout + c) * CT;
    o0[(size_t)i * N + pos] = mod_add(ca, sa, q);
    o0[(size_t)(K + i) * N + pos] = mod_add(cb, sb, q);
    if (c + C < Cout) {
      u32* o1 = out + ((size_t)b * Cout + c + C) * CT;
      o1[(size_t)i * N + pos] = csub(mul_shoup(mod_sub(ca, sa, q), w.x, w.y, q), q);
      o1[(size_t)(K + i) * N + pos] = csub(mul_shoup(mod_sub(cb, sb, q), w.x, w.y, q), q);
    }
  }
}

// (4a'') node-batched MAC with 4 consecutive slots per thread (128-bit loads and
// stores for everything but the automorphism gathers).
template <int LOGN, int K, int ELL, int NB>
__global__ void __launch_bounds__(256) k_op_eq_mac_nb4(const u32* __restrict__ state, int C, int node0, int nodes,
                                                       const u32* __restrict__ dn, RowsDesc ksk, u32 k_aut,
                                                       const uint2* __restrict__ mono, u32* __restrict__ out, int Cout,
                                                       Tables tb, int skip_c = 0) {
  constexpr int N = 1 << LOGN;
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t groups = ((size_t)nodes + NB - 1) / NB;
  if (g >= groups * K * (N / 4)) return;
  const int pos = (int)(g & (N / 4 - 1)) * 4;
  const int i = (int)((g / (N / 4)) % K);
  const int nd0 = (int)(g / ((size_t)K * (N / 4))) * NB;
  const size_t CT = 2 * (size_t)K * N;
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  u32 src_pos[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) src_pos[r] = aut_src(pos + r, k_aut, LOGN);
  int cur_b = -1;
  uint4 ka[ELL], kb[ELL];
#pragma unroll 1
  for (int u = 0; u < NB; ++u) {
    const int nd = nd0 + u;
    if (nd >= nodes) break;
    const int gn = node0 + nd;
    const int b = gn / C, c = gn % C;
    if (c < skip_c) continue;  // a row node: written by k_op_eq_mac_a8q
    if (b != cur_b) {
#pragma unroll
      for (int j = 0; j < ELL; ++j) {
        const u32* ra = ksk.row(b, j, ELL, CT) + (size_t)i * N + pos;
        ka[j] = __ldg(reinterpret_cast<const uint4*>(ra));
        kb[j] = __ldg(reinterpret_cast<const uint4*>(ra + (size_t)K * N));
      }
      cur_b = b;
    }
    const u32* st = state + (size_t)gn * CT;
    u64 a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < ELL; ++j) {  // digit ELL-1 is folded: its term is tau(a) itself
      u32 d[4];
      if (j < ELL - 1) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(dn + (((size_t)nd * ELL + j) * K + i) * N + pos));
        d[0] = v.x, d[1] = v.y, d[2] = v.z, d[3] = v.w;
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r) d[r] = __ldg(st + (size_t)i * N + src_pos[r]);
      }
      const u32 kav[4] = {ka[j].x, ka[j].y, ka[j].z, ka[j].w}, kbv[4] = {kb[j].x, kb[j].y, kb[j].z, kb[j].w};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        a0[r] += (u64)d[r] * kav[r];
        a1[r] += (u64)d[r] * kbv[r];
      }
    }
    const uint4 ca4 = __ldg(reinterpret_cast<const uint4*>(st + (size_t)i * N + pos));
    const uint4 cb4 = __ldg(reinterpret_cast<const uint4*>(st + (size_t)(K + i) * N + pos));
    const u32 ca[4] = {ca4.x, ca4.y, ca4.z, ca4.w}, cb[4] = {cb4.x, cb4.y, cb4.z, cb4.w};
    u32 xa[4], xb[4], ya[4], yb[4];
    const bool second = c + C < Cout;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const u32 sa = reduce_u64(a0[r], M);
      const u32 sb = mod_add(reduce_u64(a1[r], M), __ldg(st + (size_t)(K + i) * N + src_pos[r]), q);
      xa[r] = mod_add(ca[r], sa, q);
      xb[r] = mod_add(cb[r], sb, q);
      if (second) {
        const uint2 w = __ldg(&mono[(size_t)i * N + pos + r]);
        ya[r] = csub(mul_shoup(mod_sub(ca[r], sa, q), w.x, w.y, q), q);
        yb[r] = csub(mul_shoup(mod_sub(cb[r], sb, q), w.x, w.y, q), q);
      }
    }
    u32* o0 = out + ((size_t)b * Cout + c) * CT;
    *reinterpret_cast<uint4*>(o0 + (size_t)i * N + pos) = make_uint4(xa[0], xa[1], xa[2], xa[3]);
    *reinterpret_cast<uint4*>(o0 + (size_t)(K + i) * N + pos) = make_uint4(xb[0], xb[1], xb[2], xb[3]);
    if (second) {
      u32* o1 = out + ((size_t)b * Cout + c + C) * CT;
      *reinterpret_cast<uint4*>(o1 + (size_t)i * N + pos) = make_uint4(ya[0], ya[1], ya[2], ya[3]);
      *reinterpret_cast<uint4*>(o1 + (size_t)(K + i) * N + pos) = make_uint4(yb[0], yb[1], yb[2], yb[3]);
    }
  }
}

// Byte-plane layout of the tensor-core RowSel A operand (rowsel_tc.cuh): the
// 16-byte K group kg (depth k = 16 kg ..) of row m at slot p, plane pl lives at
// p s_p + (kg / G) s_c + (m / RA) s_mt + pl s_pl + (kg % G) s_g + (m % RA) 16.
// Rows 2b and 2b + 1 (the a and b components of query b) are adjacent 16-byte
// pieces of one core matrix, so the two components form one 32-byte sector.
struct A8Desc {
  uint8_t* base;
  size_t s_p, s_c, s_mt, s_pl, s_g;
  int G, RA;
  __device__ __forceinline__ uint8_t* at(int p, int m, int kg, int pl) const {
    return base + (size_t)p * s_p + (size_t)(kg / G) * s_c + (size_t)(m / RA) * s_mt + (size_t)pl * s_pl +
           (size_t)(kg % G) * s_g + (size_t)(m % RA) * 16;
  }
};

// (4a-v) the LAST ExpandQuery stage's MAC + combine for the row nodes (c < d0)
// with the RowSel operand pack fused in (_expanded_to_in0 + transpose_ct_tensor,
// src/protocol.py:426-441, src/layout.py:156-178), laid out for coalesced
// byte-plane writes: a warp covers 8 consecutive slots x 4 consecutive queries,
// a CTA 8 slots x 32 queries, and each thread 16 consecutive nodes (one 16-byte
// K group) of one slot.  The c + s outputs go to the A operand only -- per
// (slot, plane) the warp writes rows 2b .. 2b + 7 of one K group, 128
// contiguous bytes, the CTA 512 -- and the X^{-2^t} (c - s) outputs (c + C <
// Cout) as u32 words.  Grid: x = (N / 8) x K, y = ceil(nq / 32) over the chunk's
// queries [b0, b0 + nq), z = d0 / 16 node groups; dn holds the chunk's digit NTTs
// with node index (b - b0) C + c.  Requires d0 % 16 == 0 and d0 <= C.
template <int LOGN, int K, int ELL>
__global__ void __launch_bounds__(256) k_op_eq_mac_a8q(const u32* __restrict__ state, int C, int b0, int nq,
                                                       const u32* __restrict__ dn, RowsDesc ksk, u32 k_aut,
                                                       const uint2* __restrict__ mono, u32* __restrict__ out, int Cout,
                                                       Tables tb, A8Desc a8) {
  constexpr int N = 1 << LOGN;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pos = (int)(blockIdx.x % (N / 8)) * 8 + (lane & 7);
  const int i = (int)(blockIdx.x / (N / 8));
  const int bl = (int)blockIdx.y * 32 + warp * 4 + (lane >> 3);
  if (bl >= nq) return;
  const int b = b0 + bl, c0 = (int)blockIdx.z * 16;
  const size_t CT = 2 * (size_t)K * N;
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  const u32 src_pos = aut_src(pos, k_aut, LOGN);
  const uint2 w = __ldg(&mono[(size_t)i * N + pos]);
  u32 ka[ELL], kb[ELL];
#pragma unroll
  for (int j = 0; j < ELL; ++j) {
    const u32* ra = ksk.row(b, j, ELL, CT) + (size_t)i * N + pos;
    ka[j] = __ldg(ra);
    kb[j] = __ldg(ra + (size_t)K * N);
  }
  u32 pa[4][4], pb[4][4];  // [plane][word]: byte u of the 16-byte K group = node c0 + u
#pragma unroll
  for (int pl = 0; pl < 4; ++pl)
#pragma unroll
    for (int v = 0; v < 4; ++v) pa[pl][v] = pb[pl][v] = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int c = c0 + u;
    const size_t nd = (size_t)bl * C + c;
    const u32* st = state + ((size_t)b * C + c) * CT;
    u64 a0 = 0, a1 = 0;
#pragma unroll
    for (int j = 0; j < ELL; ++j) {  // digit ELL-1 is folded: its term is tau(a) itself
      const u32 d = j < ELL - 1 ? __ldg(dn + ((nd * ELL + j) * K + i) * N + pos) : __ldg(st + (size_t)i * N + src_pos);
      a0 += (u64)d * ka[j];
      a1 += (u64)d * kb[j];
    }
    const u32 ca = __ldg(st + (size_t)i * N + pos), cb = __ldg(st + (size_t)(K + i) * N + pos);
    const u32 sa = reduce_u64(a0, M);
    const u32 sb = mod_add(reduce_u64(a1, M), __ldg(st + (size_t)(K + i) * N + src_pos), q);
    const u32 xa = mod_add(ca, sa, q), xb = mod_add(cb, sb, q);
#pragma unroll
    for (int pl = 0; pl < 4; ++pl) {
      pa[pl][u >> 2] |= ((xa >> (8 * pl)) & 0xffu) << (8 * (u & 3));
      pb[pl][u >> 2] |= ((xb >> (8 * pl)) & 0xffu) << (8 * (u & 3));
    }
    if (c + C < Cout) {
      u32* o1 = out + ((size_t)b * Cout + c + C) * CT;
      o1[(size_t)i * N + pos] = csub(mul_shoup(mod_sub(ca, sa, q), w.x, w.y, q), q);
      o1[(size_t)(K + i) * N + pos] = csub(mul_shoup(mod_sub(cb, sb, q), w.x, w.y, q), q);
    }
  }
  const int p = i * N + pos, kg = c0 >> 4;
#pragma unroll
  for (int pl = 0; pl < 4; ++pl) {
    uint4* d = reinterpret_cast<uint4*>(a8.at(p, 2 * b, kg, pl));  // rows 2b, 2b + 1: one 32-byte sector
    d[0] = make_uint4(pa[pl][0], pa[pl][1], pa[pl][2], pa[pl][3]);
    d[1] = make_uint4(pb[pl][0], pb[pl][1], pb[pl][2], pb[pl][3]);
  }
}

// (4b) external-product MAC (+ ColTor combine); one thread per (ct, limb, slot).
template <int LOGN, int K, int ELL>
__global__ void k_op_xp_mac(const u32* __restrict__ in, size_t in_b, int M_per_b, int m0, int cts, int pairs,
                            const u32* __restrict__ dn, RowsDesc rows, u32* __restrict__ out, size_t out_b, Tables tb) {
  constexpr int N = 1 << LOGN;
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (size_t)cts * K * N) return;
  const int pos = (int)(g & (N - 1));
  const int i = (int)((g >> LOGN) % K);
  const int ct = (int)(g / ((size_t)K * N));
  const int gm = m0 + ct;
  const int b = gm / M_per_b, m = gm % M_per_b;
  const size_t CT = 2 * (size_t)K * N;
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  const u32* src = pairs ? in + (b * in_b + 2 * (size_t)m) * CT : in + (b * in_b + (size_t)m) * CT;
  u64 a0 = 0, a1 = 0;
#pragma unroll
  for (int comp = 0; comp < 2; ++comp) {
#pragma unroll
    for (int j = 0; j < ELL; ++j) {
      u32 d;
      if (j < ELL - 1) {
        d = __ldg(dn + ((((size_t)ct * 2 + comp) * ELL + j) * K + i) * N + pos);
      } else {  // folded top digit: this component of the input (or odd - even)
        const size_t off = (size_t)(comp * K + i) * N + pos;
        d = pairs ? pair_diff1(src, off, pairs, CT, q) : __ldg(src + off);
      }
      const u32* ra = rows.row(b, comp * ELL + j, ELL, CT) + (size_t)i * N + pos;
      a0 += (u64)d * __ldg(ra);
      a1 += (u64)d * __ldg(ra + (size_t)K * N);
    }
  }
  u32 sa = reduce_u64(a0, M), sb = reduce_u64(a1, M);
  if (pairs) {
    const u32* ev = in + (b * in_b + 2 * (size_t)m) * CT;
    sa = mod_add(sa, pair_even1(ev, (size_t)i * N + pos, pairs), q);
    sb = mod_add(sb, pair_even1(ev, (size_t)(K + i) * N + pos, pairs), q);
  }
  u32* d = out + (b * out_b + (size_t)m) * CT;
  d[(size_t)i * N + pos] = sa;
  d[(size_t)(K + i) * N + pos] = sb;
}

// (4b') the same with NB consecutive ciphertexts per thread: the cts of one query
// (the ColTor pairs of one level, the RGSW-assembly column cts) share their key
// rows, loaded once per group and reloaded only where it crosses into the next query.
template <int LOGN, int K, int ELL, int NB>
__global__ void k_op_xp_mac_nb(const u32* __restrict__ in, size_t in_b, int M_per_b, int m0, int cts, int pairs,
                               const u32* __restrict__ dn, RowsDesc rows, u32* __restrict__ out, size_t out_b,
                               Tables tb) {
  constexpr int N = 1 << LOGN;
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t groups = ((size_t)cts + NB - 1) / NB;
  if (g >= groups * K * N) return;
  const int pos = (int)(g & (N - 1));
  const int i = (int)((g >> LOGN) % K);
  const int ct0 = (int)(g / ((size_t)K * N)) * NB;
  const size_t CT = 2 * (size_t)K * N;
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  int cur_b = -1;
  u32 ka[2 * ELL], kb[2 * ELL];
#pragma unroll 1
  for (int u = 0; u < NB; ++u) {
    const int ct = ct0 + u;
    if (ct >= cts) break;
    const int gm = m0 + ct;
    const int b = gm / M_per_b, m = gm % M_per_b;
    if (b != cur_b) {
#pragma unroll
      for (int r = 0; r < 2 * ELL; ++r) {
        const u32* ra = rows.row(b, r, ELL, CT) + (size_t)i * N + pos;
        ka[r] = __ldg(ra);
        kb[r] = __ldg(ra + (size_t)K * N);
      }
      cur_b = b;
    }
    const u32* src = pairs ? in + (b * in_b + 2 * (size_t)m) * CT : in + (b * in_b + (size_t)m) * CT;
    u64 a0 = 0, a1 = 0;
#pragma unroll
    for (int comp = 0; comp < 2; ++comp) {
#pragma unroll
      for (int j = 0; j < ELL; ++j) {
        u32 d;
        if (j < ELL - 1) {
          d = __ldg(dn + ((((size_t)ct * 2 + comp) * ELL + j) * K + i) * N + pos);
        } else {  // folded top digit: this component of the input (or odd - even)
          const size_t off = (size_t)(comp * K + i) * N + pos;
          d = pairs ? pair_diff1(src, off, pairs, CT, q) : __ldg(src + off);
        }
        a0 += (u64)d * ka[comp * ELL + j];
        a1 += (u64)d * kb[comp * ELL + j];
      }
    }
    u32 sa = reduce_u64(a0, M), sb = reduce_u64(a1, M);
    if (pairs) {
      const u32* ev = in + (b * in_b + 2 * (size_t)m) * CT;
      sa = mod_add(sa, pair_even1(ev, (size_t)i * N + pos, pairs), q);
      sb = mod_add(sb, pair_even1(ev, (size_t)(K + i) * N + pos, pairs), q);
    }
    u32* d = out + (b * out_b + (size_t)m) * CT;
    d[(size_t)i * N + pos] = sa;
    d[(size_t)(K + i) * N + pos] = sb;
  }
}

// (4b'') node-batched external-product MAC with 4 consecutive slots per thread.
template <int LOGN, int K, int ELL, int NB>
__global__ void __launch_bounds__(256) k_op_xp_mac_nb4(const u32* __restrict__ in, size_t in_b, int M_per_b, int m0,
                                                       int cts, int pairs, const u32* __restrict__ dn, RowsDesc rows,
                                                       u32* __restrict__ out, size_t out_b, Tables tb) {
  constexpr int N = 1 << LOGN;
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t groups = ((size_t)cts + NB - 1) / NB;
  if (g >= groups * K * (N / 4)) return;
  const int pos = (int)(g & (N / 4 - 1)) * 4;
  const int i = (int)((g / (N / 4)) % K);
  const int ct0 = (int)(g / ((size_t)K * (N / 4))) * NB;
  const size_t CT = 2 * (size_t)K * N;
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  int cur_b = -1;
  uint4 ka[2 * ELL], kb[2 * ELL];
#pragma unroll 1
  for (int u = 0; u < NB; ++u) {
    const int ct = ct0 + u;
    if (ct >= cts) break;
    const int gm = m0 + ct;
    const int b = gm / M_per_b, m = gm % M_per_b;
    if (b != cur_b) {
#pragma unroll
      for (int r = 0; r < 2 * ELL; ++r) {
        const u32* ra = rows.row(b, r, ELL, CT) + (size_t)i * N + pos;
        ka[r] = __ldg(reinterpret_cast<const uint4*>(ra));
        kb[r] = __ldg(reinterpret_cast<const uint4*>(ra + (size_t)K * N));
      }
      cur_b = b;
    }
    const u32* src = pairs ? in + (b * in_b + 2 * (size_t)m) * CT : in + (b * in_b + (size_t)m) * CT;
    u64 a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0};
#pragma unroll
    for (int comp = 0; comp < 2; ++comp) {
#pragma unroll
      for (int j = 0; j < ELL; ++j) {
        uint4 v;
        if (j < ELL - 1) {
          v = __ldg(reinterpret_cast<const uint4*>(dn + ((((size_t)ct * 2 + comp) * ELL + j) * K + i) * N + pos));
        } else {  // folded top digit: this component of the input (or odd - even)
          const size_t off = (size_t)(comp * K + i) * N + pos;
          if (pairs) {
            uint4 o;
            pair_ld4(src, off, pairs, CT, v, o);
            v = make_uint4(mod_sub(o.x, v.x, q), mod_sub(o.y, v.y, q), mod_sub(o.z, v.z, q), mod_sub(o.w, v.w, q));
          } else {
            v = __ldg(reinterpret_cast<const uint4*>(src + off));
          }
        }
        const uint4 kr = ka[comp * ELL + j], ks = kb[comp * ELL + j];
        a0[0] += (u64)v.x * kr.x, a0[1] += (u64)v.y * kr.y, a0[2] += (u64)v.z * kr.z, a0[3] += (u64)v.w * kr.w;
        a1[0] += (u64)v.x * ks.x, a1[1] += (u64)v.y * ks.y, a1[2] += (u64)v.z * ks.z, a1[3] += (u64)v.w * ks.w;
      }
    }
    u32 sa[4], sb[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) sa[r] = reduce_u64(a0[r], M), sb[r] = reduce_u64(a1[r], M);
    if (pairs) {
      const u32* ev = in + (b * in_b + 2 * (size_t)m) * CT;
      const uint4 ea = pair_even4(ev, (size_t)i * N + pos, pairs);
      const uint4 eb = pair_even4(ev, (size_t)(K + i) * N + pos, pairs);
      sa[0] = mod_add(sa[0], ea.x, q), sa[1] = mod_add(sa[1], ea.y, q), sa[2] = mod_add(sa[2], ea.z, q),
      sa[3] = mod_add(sa[3], ea.w, q);
      sb[0] = mod_add(sb[0], eb.x, q), sb[1] = mod_add(sb[1], eb.y, q), sb[2] = mod_add(sb[2], eb.z, q),
      sb[3] = mod_add(sb[3], eb.w, q);
    }
    u32* d = out + (b * out_b + (size_t)m) * CT;
    *reinterpret_cast<uint4*>(d + (size_t)i * N + pos) = make_uint4(sa[0], sa[1], sa[2], sa[3]);
    *reinterpret_cast<uint4*>(d + (size_t)(K + i) * N + pos) = make_uint4(sb[0], sb[1], sb[2], sb[3]);
  }
}

// ---------------------------------------------------------------------------
// RowSel on CUDA cores (row_select_raw, src/protocol.py:448-492): 4N
// independent mod-q GEMMs over the p axis, out[b, j, comp, p] =
// sum_i rows[b, i, comp, p] * db[j, i, p] mod q(p).  P-major operands (p
// contiguous), one warp lane per p, a CTA covers 32 p x (MT x NT) outputs
// and streams K in double-buffered cp.async chunks; products accumulate in
// 64 bits and are folded mod q every 1024 terms (the reference's _k_chunk,
// src/layout.py:185-187).
constexpr int RS_MT = 16, RS_NT = 16, RS_KC = 8;
constexpr int RS_SMEM = 2 * RS_KC * (RS_MT + RS_NT) * 32 * 4;

__device__ __forceinline__ void cp_async16(void* smem_ptr, const void* gptr, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_ptr);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gptr), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NWAIT>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NWAIT));
}

__global__ void __launch_bounds__(256)
    k_rowsel_cc(const u32* __restrict__ A, size_t a_b /* words per query */, int Mrows /* 2B */,
                const u32* __restrict__ db, int d0, int d1, u32* __restrict__ out, int KN, int logn, Tables tb) {
  extern __shared__ __align__(16) u32 rs_smem[];
  u32(*As)[RS_KC][RS_MT][32] = reinterpret_cast<u32(*)[RS_KC][RS_MT][32]>(rs_smem);
  u32(*Ds)[RS_KC][RS_NT][32] = reinterpret_cast<u32(*)[RS_KC][RS_NT][32]>(rs_smem + 2 * RS_KC * RS_MT * 32);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mtiles = (Mrows + RS_MT - 1) / RS_MT;
  const int mt = blockIdx.x % mtiles, nt = blockIdx.x / mtiles;
  const int p0 = blockIdx.y * 32;
  const int m0 = mt * RS_MT, n0 = nt * RS_NT;
  const Modulus M = tb.mod[p0 >> logn];
  const int mg = warp & 3, ng = warp >> 2;  // thread tile: 4 m x 8 n
  u64 acc[4][8];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[t][u] = 0;

  auto issue = [&](int stage, int k0) {
    // A tile: RS_KC x RS_MT rows of 32 words (8 x 16B chunks each) = 1024 chunks
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int ch = tid + it * 256;
      const int row = ch >> 3, part = ch & 7;
      const int kk = row / RS_MT, mm = row % RS_MT;
      const int m = m0 + mm, kidx = k0 + kk;
      const bool ok = m < Mrows && kidx < d0;
      const int b = m >> 1, comp = m & 1;
      const u32* g = A + (ok ? (size_t)b * a_b + ((size_t)kidx * 2 + comp) * KN + p0 + part * 4 : 0);
      cp_async16(&As[stage][kk][mm][part * 4], ok ? g : A, ok);
    }
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int ch = tid + it * 256;
      const int row = ch >> 3, part = ch & 7;
      const int kk = row / RS_NT, nn = row % RS_NT;
      const int n = n0 + nn, kidx = k0 + kk;
      const bool ok = n < d1 && kidx < d0;
      const u32* g = db + (ok ? ((size_t)n * d0 + kidx) * KN + p0 + part * 4 : 0);
      cp_async16(&Ds[stage][kk][nn][part * 4], ok ? g : db, ok);
    }
    cp_async_commit();
  };

  const int nk = (d0 + RS_KC - 1) / RS_KC;
  issue(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc & 1;
    if (kc + 1 < nk) {
      issue(s ^ 1, (kc + 1) * RS_KC);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < RS_KC; ++kk) {
      u32 a[4], d[8];
#pragma unroll
      for (int t = 0; t < 4; ++t) a[t] = As[s][kk][mg * 4 + t][lane];
#pragma unroll
      for (int u = 0; u < 8; ++u) d[u] = Ds[s][kk][ng * 8 + u][lane];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[t][u] += (u64)a[t] * d[u];
    }
    if (((kc + 1) * RS_KC) % 1024 == 0) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[t][u] = reduce_u64(acc[t][u], M);
    }
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int m = m0 + mg * 4 + t;
    if (m >= Mrows) continue;
    const int b = m >> 1, comp = m & 1;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int n = n0 + ng * 8 + u;
      if (n >= d1) continue;
      out[(((size_t)b * d1 + n) * 2 + comp) * KN + p0 + lane] = reduce_u64(acc[t][u], M);
    }
  }
}

// ---------------------------------------------------------------------------
// DB preprocessing (encode_database, src/protocol.py:118-153): record bytes
// -> little-endian base-P words -> centered mod P -> lifted mod q_i ->
// forward NTT, written straight into the GPU P-major brv layout
// db[j][i][limb][slot].  grid (records, K).
template <int LOGN, int K>
__global__ void __launch_bounds__(NttCfg<LOGN>::T)
    k_db_encode(const uint8_t* __restrict__ recs, int rec_bytes, int d0, int d1, int plain_bits,
                u32* __restrict__ db, Tables tb, const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN;
  __shared__ __align__(16) u32 xbuf[2 * N];
  NttState ns{xbuf, 0};
  const int r = blockIdx.x, i = blockIdx.y;
  const int row = r / d1, col = r % d1;
  const uint8_t* rec = recs + (size_t)r * rec_bytes;
  const int width = plain_bits / 8;
  const u32 q = tb.mod[i].q;
  u32* dst = db + (((size_t)col * d0 + row) * K + i) * N;
  ntt_fwd<LOGN>(
      ns, tb.fwd + (size_t)i * N, tc.f[i], tb.mod[i],
      [&](int j) -> u32 {
        u64 w = 0;
        for (int t = 0; t < width; ++t) {
          const int o = j * width + t;
          if (o < rec_bytes) w |= (u64)__ldg(rec + o) << (8 * t);
        }
        // center into [-P/2, P/2) then lift (src/protocol.py:145-147)
        const u64 P = 1ull << plain_bits;
        if (w >= (P >> 1)) {
          const u64 neg = P - w;  // |m|, at most P/2 <= 2^31
          return (u32)((q - (u32)(neg % q)) % q);
        }
        return (u32)(w % q);
      },
      [&](int i0, const u32(&x)[16]) { st16(dst + i0, x); });
}

// In-place reduction of limb rows holding sums of up to 16 canonical residues
// (the NCCL modular-add combine of row-sharded RowSel partials).
__global__ void k_mod_rows(u32* __restrict__ x, size_t rows, int logn, int k, Tables tb) {
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (rows << logn)) return;
  const int limb = (int)((g >> logn) % k);
  const Modulus& M = tb.mod[limb];
  x[g] = x[g] % M.q;
}

// Bit-reversal permutation of whole limb rows (natural <-> brv; an involution).
// out[r][p] = in[p][r] for a P x R u32 matrix (32 x 32 tiles through shared memory)
__global__ void k_transpose32(const u32* __restrict__ in, u32* __restrict__ out, size_t P, size_t R) {
  __shared__ u32 t[32][33];
  const size_t r0 = (size_t)blockIdx.x * 32, p0 = (size_t)blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += 8)
    if (p0 + y < P && r0 + threadIdx.x < R) t[y][threadIdx.x] = in[(p0 + y) * R + r0 + threadIdx.x];
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8)
    if (r0 + y < R && p0 + threadIdx.x < P) out[(r0 + y) * P + p0 + threadIdx.x] = t[threadIdx.x][y];
}

__global__ void k_bitrev_rows(const u32* __restrict__ in, u32* __restrict__ out, size_t rows, int logn) {
  const size_t n = (size_t)1 << logn;
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= rows * n) return;
  const size_t row = g >> logn;
  const u32 j = (u32)(g & (n - 1));
  out[g] = __ldg(in + row * n + brv(j, logn));
}

}  // namespace gpir
