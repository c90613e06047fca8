// Shared device definitions for the GPIR server pipeline on sm_100a.
//
// Data convention: every NTT-domain polynomial
// limb lives in HBM as n uint32 canonical residues in BIT-REVERSED slot order
// ("brv layout"): position i holds the evaluation ntt(a)[brv(i)] of the
// reference's natural-order transform (src/ring.py:6-12).  With that layout the
// forward transform is a plain Cooley-Tukey DIT (natural coeffs -> brv) and
// the inverse a Gentleman-Sande DIF (brv -> natural coeffs), so no transform
// ever permutes through HBM.  Conversion to/from the reference's natural
// order happens only at the C-ABI boundary.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gpir {

typedef uint32_t u32;
typedef uint64_t u64;

constexpr int kMaxLimbs = 8;
constexpr int kMaxEll = 16;

// Per-limb modulus constants.
struct Modulus {
  u32 q;
  u32 qinv_neg;   // -q^{-1} mod 2^32 (Montgomery REDC)
  u32 r2;         // 2^64 mod q  (REDC(hi * r2) = hi * 2^32 mod q)
  u32 barrett;    // floor(2^32 / q)
  u32 ninv;       // n^{-1} mod q
  u32 ninv_sh;    // Shoup companion of ninv
  u32 mhat;       // (Q/q)^{-1} mod q   (CRT, src/ring.py:216-220)
  u32 mhat_sh;
  u32 r1;         // 2^32 mod q (undoes the Montgomery factor of mont_mac)
  u32 r1_sh;
};

// CRT / gadget constants (src/ring.py:214-235, src/he.py:45-55).
struct CrtConst {
  int k;
  int ell;
  int z_bits;
  int logn;
  u64 m_lo[kMaxLimbs], m_hi[kMaxLimbs];   // Q / q_i as 128-bit
  u64 q_lo, q_hi;                         // Q
  u64 half_lo, half_hi;                   // (Q-1)/2
  int n_red;                              // descending multiples t*Q to subtract
  u64 red_lo[4], red_hi[4];
  u64 dc_lo, dc_hi;                       // sum_{j < ell-1} (z/2 - 1) z^j (closed-form digits)
};

// Top-digit fold constants (see k_fold_rows): per limb i, w[i][j] = z^(j-(ell-1))
// mod q_i for j < ell-1 and w[i][ell-1] = z^-(ell-1), with Shoup companions.
struct FoldConst {
  uint2 w[kMaxLimbs][kMaxEll];
};

// Device-resident transform tables for one context.
struct Tables {
  const uint2* fwd;    // [k][n] (psi^brv(i), shoup)     forward CT twiddles
  const uint2* inv;    // [k][n] (psi^-brv(i), shoup)    inverse GS twiddles
  Modulus mod[kMaxLimbs];
};

__device__ __forceinline__ u32 mulhi(u32 a, u32 b) { return __umulhi(a, b); }

// x * w mod q lazily in [0, 2q) for any 32-bit x (Shoup).
__device__ __forceinline__ u32 mul_shoup(u32 x, u32 w, u32 wsh, u32 q) {
  return x * w - mulhi(x, wsh) * q;
}

// x < 2m <= 2^32 -> x mod m as an unsigned min (one ALU VIMNMX instead of
// ISETP + SEL): if x < m, x - m wraps above x.
__device__ __forceinline__ u32 csub(u32 x, u32 m) { return min(x, x - m); }

// Montgomery REDC: u < q * 2^32  ->  u * 2^-32 mod q in [0, 2q).
__device__ __forceinline__ u32 redc(u64 u, const Modulus& M) {
  u32 m = (u32)u * M.qinv_neg;
  return (u32)((u + (u64)m * M.q) >> 32);
}

// Any 64-bit value mod q, canonical.
__device__ __forceinline__ u32 reduce_u64(u64 x, const Modulus& M) {
  u32 hi = (u32)(x >> 32), lo = (u32)x;
  u32 a = redc((u64)hi * M.r2, M);                // hi * 2^32 mod q, [0, 2q)
  u32 b = lo - mulhi(lo, M.barrett) * M.q;        // lo mod q, [0, 2q)
  u32 r = a + b;                                   // [0, 4q)
  r = csub(r, 2 * M.q);
  return csub(r, M.q);
}

// 64-bit MAC accumulator as two independent 32-bit registers.  u64 register
// pairs must be even-aligned, which inside the NTT loops costs ~100 register
// moves per transform; the explicit carry chain (IMAD + IMAD.HI.X) does not.
struct Acc {
  u32 lo, hi;
};

__device__ __forceinline__ void acc_zero(Acc& a) { a.lo = a.hi = 0; }

__device__ __forceinline__ void acc_mac(Acc& a, u32 x, u32 y) {
  asm("{\n\t.reg .u32 h;\n\tmul.hi.u32 h, %2, %3;\n\tmad.lo.cc.u32 %0, %2, %3, %0;\n\taddc.u32 %1, %1, h;\n\t}"
      : "+r"(a.lo), "+r"(a.hi)
      : "r"(x), "r"(y));
}

__device__ __forceinline__ u32 mod_add(u32 a, u32 b, u32 q) { return csub(a + b, q); }

// Signed lazy Montgomery MAC: acc += x*y*2^-32 mod q, exactly representable:
// with m = lo(x*y) * q^-1 mod 2^32 the low words of x*y and m*q agree, so
// (x*y - m*q) / 2^32 = hi(x*y) - hi(m*q), which lies in (-q, q) for any
// 32-bit x and y < q.  Four IMAD-class ops and a 32-bit accumulator (no
// 64-bit register pairs); `terms` such products stay in int32 while
// terms * q < 2^31.
#ifndef MONT_WIDE
#define MONT_WIDE 1
#endif
__device__ __forceinline__ void mont_mac(int& acc, u32 x, u32 y, u32 q, u32 qinv) {
#if MONT_WIDE  // one IMAD.WIDE (quarter rate) for both halves instead of IMAD + IMAD.HI
  const u64 p = (u64)x * y;
  const u32 lo = (u32)p, hi = (u32)(p >> 32);
#else
  const u32 lo = x * y, hi = __umulhi(x, y);
#endif
  acc += (int)(hi - __umulhi(lo * qinv, q));
}

// canonical (acc * 2^32) mod q for an accumulator of `terms` mont_mac terms
__device__ __forceinline__ u32 mont_fin(int acc, int terms, const Modulus& M) {
  const u32 v = (u32)(acc + terms * (int)M.q);  // in (0, 2 terms q)
  return csub(mul_shoup(v, M.r1, M.r1_sh, M.q), M.q);
}

__device__ __forceinline__ u32 reduce_acc(const Acc& a, const Modulus& M) {
  return reduce_u64(((u64)a.hi << 32) | a.lo, M);
}
__device__ __forceinline__ u32 mod_sub(u32 a, u32 b, u32 q) { return csub(a + q - b, q); }

__device__ __forceinline__ u32 mod_mul(u32 a, u32 b, const Modulus& M) {
  return reduce_u64((u64)a * b, M);
}

__device__ __forceinline__ u32 brv(u32 x, int logn) { return __brev(x) >> (32 - logn); }

// Automorphism X -> X^k_aut as a gather on the brv layout:
// natural P[j] = (((2j+1) k mod 2n) - 1)/2  (src/ring.py:643-654)
// brv:  out[i] = in[brv(P[brv(i)])].
__device__ __forceinline__ u32 aut_src(u32 i, u32 k_aut, int logn) {
  u32 j = brv(i, logn);
  u32 two_n_mask = (2u << logn) - 1;
  u32 e = ((2 * j + 1) * k_aut) & two_n_mask;
  return brv((e - 1) >> 1, logn);
}

}  // namespace gpir
