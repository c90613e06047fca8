// Block-level negacyclic NTT / inverse NTT for one polynomial limb.
//
// One CTA of T = n/16 threads owns one n-point limb; every thread holds 16
// elements in registers.  The forward transform is Cooley-Tukey DIT with the
// psi twist merged into bit-reversed twiddles (natural coeffs -> brv evals);
// the inverse is Gentleman-Sande DIF (brv evals -> natural coeffs) with the
// n^{-1} scale applied at the end.  Both compute exactly the reference's
// transform (src/ring.py:408-453) up to the slot permutation documented in
// gpir_common.cuh.  Products are 32-bit Shoup; the forward transform is fully
// lazy (values grow < 2q per stage, reduced once at the end — the reference's
// numba kernel uses the same bound, src/ring.py:320-374), the inverse keeps
// Harvey's [0, 2q) invariant.
//
// For n = 2^LOGN with LOGN % 4 == 0 the transform runs as LOGN/4 radix-16
// passes over registers with shared-memory exchanges.  Of the two exchanges
// of an n = 4096 transform one is block-wide and one stays inside a warp
// (the warp's 512 elements are the same set in both passes), so a transform
// costs ONE block barrier.  xbuf holds two n-word buffers; consecutive
// transforms alternate between them (`NttState::parity`), which makes a
// single barrier per transform race-free.  The swizzled layout keeps all
// three access patterns bank-conflict free at n = 4096.  Twiddles of the
// passes whose butterfly bits are >= 4 (table index < 256) come from kernel
// parameter space (__grid_constant__, constant cache); the per-thread runs of
// the last pass are read from the global table with 128-bit loads.  Other
// sizes (the tiny test rings) use a shared-memory radix-2 loop with the same
// I/O contract.
//
// I/O contract (both paths):
//   forward: ld(j) is called for natural coefficient j = tid | r << (LOGN-4)
//            (r = 0..15);  st(i0, x[16]) receives brv slots i0 = 16*tid + r.
//   inverse: ld16(i0, x[16]) must fill brv slots i0 = 16*tid + r;
//            st(j, r, v) receives natural coefficient j = tid | r << (LOGN-4).
//   `stage_buffer(ns)` is free for the caller to stage the NEXT transform's
//   inputs (after a block barrier).
#pragma once
#include "gpir_common.cuh"

namespace gpir {

constexpr int kTwConstEntries = 256;
constexpr int kTwConstLimbs = 4;

// twiddle entries with table index < 256, per limb, fwd and inv
struct TwConst {
  uint2 f[kTwConstLimbs][kTwConstEntries];
  uint2 i[kTwConstLimbs][kTwConstEntries];
};

template <int LOGN>
struct NttCfg {
  static constexpr int N = 1 << LOGN;
  static constexpr int T = N / 16;
  static constexpr bool kFast = (LOGN % 4 == 0) && LOGN >= 8;
  static constexpr int SHIFT = LOGN - 4;
  static constexpr int XBUF_WORDS = 2 * N;
};

struct NttState {
  u32* xbuf;   // 2 * n words
  int parity;  // buffer of the next transform
};

template <int LOGN>
__device__ __forceinline__ u32* stage_buffer(const NttState& ns) {
  return ns.xbuf + (ns.parity ^ 1) * (1 << LOGN);
}

template <int LOGN>
__device__ __forceinline__ int swz(int j) {
  if constexpr (LOGN == 12) {
    int row = j >> 5;
    return j ^ ((row & 15) ^ (((row >> 3) & 1) << 4));
  } else {
    return j;
  }
}

// element index of register r in the pass whose butterfly bits are [B0, B0+4)
template <int B0>
__device__ __forceinline__ int pidx(int tid, int r) {
  return ((tid >> B0) << (B0 + 4)) | (r << B0) | (tid & ((1 << B0) - 1));
}

// Shared-memory word address of register r for pass B0: swz(pidx(tid, r)),
// written so that per-thread parts are computed once and r only adds
// immediates (n = 4096; see the derivation in DESIGN.md "NTT exchange").
template <int LOGN, int B0>
struct XAddr {
  int base, p0, p1;
  __device__ __forceinline__ XAddr(int tid) {
    if constexpr (LOGN == 12 && B0 == 8) {
      base = tid & ~31;
      p0 = (tid & 31) ^ (tid >> 5);
      p1 = p0 ^ 24;
    } else if constexpr (LOGN == 12 && B0 == 4) {
      const int h = (tid >> 4) & 1;
      base = (tid >> 4) << 8;
      p0 = (tid & 15) ^ (h << 3) ^ (h << 4);
      p1 = 0;
    } else if constexpr (LOGN == 12 && B0 == 0) {
      const int row = tid >> 1;
      const int F = (row & 15) ^ (((row >> 3) & 1) << 4);
      base = row << 5;
      p0 = ((tid & 1) << 4) ^ F;
      p1 = 0;
    } else {
      base = tid;
      p0 = p1 = 0;
    }
  }
  __device__ __forceinline__ int operator()(int tid, int r) const {
    if constexpr (LOGN == 12 && B0 == 8) {
      return base + (r << 8) + ((r & 1) ? p1 : p0);
    } else if constexpr (LOGN == 12 && B0 == 4) {
      return base + ((r >> 1) << 5) + (p0 ^ (((r & 1) << 4) ^ (r >> 1)));
    } else if constexpr (LOGN == 12 && B0 == 0) {
      return base + (p0 ^ r);
    } else {
      return swz<LOGN>(pidx<B0>(tid, r));
    }
  }
};

// Twiddles of one butterfly stage.  In the pass with butterfly bits
// [B0, B0+4) and r-bit rb, the group index of register r is
//   ((tid >> B0) << (3 - rb)) + (r >> (rb + 1)),
// so a thread needs 2^(3-rb) consecutive table entries from a
// thread-dependent base.  For B0 == 0 those runs are disjoint per lane and
// 64-byte aligned: fetched with 128-bit loads.
template <int B0, int RB>
__device__ __forceinline__ void load_tw(const uint2* __restrict__ base, uint2 (&w)[8]) {
  constexpr int CNT = 1 << (3 - RB);
  if constexpr (B0 == 0 && CNT >= 2) {
    const uint4* v = reinterpret_cast<const uint4*>(base);
#pragma unroll
    for (int c = 0; c < CNT / 2; ++c) {
      const uint4 t = __ldg(v + c);
      w[2 * c] = make_uint2(t.x, t.y);
      w[2 * c + 1] = make_uint2(t.z, t.w);
    }
  } else if constexpr (B0 == 0) {
    w[0] = __ldg(base);
  } else {
#pragma unroll
    for (int c = 0; c < CNT; ++c) w[c] = base[c];  // parameter space (constant cache)
  }
}

template <int LOGN, int B0>
__device__ __forceinline__ int tpart(int tid) {
  return (B0 == LOGN - 4) ? 0 : (tid >> B0);  // tid < 2^(LOGN-4)
}

template <int LOGN, int B0, int RB>
__device__ __forceinline__ void fwd_stage(u32 (&x)[16], int tid, const uint2* __restrict__ twg,
                                          const uint2* twc, u32 q) {
  constexpr int S = LOGN - 1 - (B0 + RB);
  uint2 w[8];
  const int off = (1 << S) + (tpart<LOGN, B0>(tid) << (3 - RB));
  load_tw<B0, RB>((B0 == 0 ? twg : twc) + off, w);
  const u32 q2 = 2 * q;
  const u32 zero = q >> 31;  // 0 (q < 2^31), opaque to the compiler
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    if (r & (1 << RB)) continue;
    const uint2 ww = w[r >> (RB + 1)];
    const u32 u = x[r];
    const u32 t = mul_shoup(x[r | (1 << RB)], ww.x, ww.y, q);
    // u + t as max(u + t, 0): keeps the add on the ALU pipe (VIADDMNMX)
    // instead of an IMAD.IADD competing with the multiplies for the FMA pipe
    x[r] = __viaddmax_u32(u, t, zero);
    x[r | (1 << RB)] = u + q2 - t;
  }
}

template <int LOGN, int B0, int RB>
__device__ __forceinline__ void inv_stage(u32 (&x)[16], int tid, const uint2* __restrict__ twg,
                                          const uint2* twc, u32 q) {
  constexpr int U = B0 + RB;
  uint2 w[8];
  const int off = (1 << (LOGN - 1 - U)) + (tpart<LOGN, B0>(tid) << (3 - RB));
  load_tw<B0, RB>((B0 == 0 ? twg : twc) + off, w);
  const u32 q2 = 2 * q;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    if (r & (1 << RB)) continue;
    const uint2 ww = w[r >> (RB + 1)];
    const u32 a = x[r], b = x[r | (1 << RB)];
    x[r] = csub(a + b, q2);
    x[r | (1 << RB)] = mul_shoup(a + q2 - b, ww.x, ww.y, q);
  }
}

template <int LOGN, int B0>
__device__ __forceinline__ void xchg_store(u32* buf, const u32 (&x)[16], int tid) {
  const XAddr<LOGN, B0> a(tid);
#pragma unroll
  for (int r = 0; r < 16; ++r) buf[a(tid, r)] = x[r];
}

template <int LOGN, int B0>
__device__ __forceinline__ void xchg_load(const u32* buf, u32 (&x)[16], int tid) {
  const XAddr<LOGN, B0> a(tid);
#pragma unroll
  for (int r = 0; r < 16; ++r) x[r] = buf[a(tid, r)];
}

// is the exchange between the passes with butterfly bits B0 and B0-4 local to
// a warp?  (both passes give a warp the same 512-element set when the lower
// pass is B0 - 4 == 0: warp w owns j in [512 w, 512 w + 512))
template <int LOGN, int BLO>
constexpr bool warp_local() {
  return BLO == 0 && LOGN == 12;
}

// ---------------------------------------------------------------------------
// forward

template <int LOGN, int B0>
__device__ __forceinline__ void fwd_passes(u32* buf, u32 (&x)[16], int tid, const uint2* twg, const uint2* twc,
                                           u32 q) {
  fwd_stage<LOGN, B0, 3>(x, tid, twg, twc, q);
  fwd_stage<LOGN, B0, 2>(x, tid, twg, twc, q);
  fwd_stage<LOGN, B0, 1>(x, tid, twg, twc, q);
  fwd_stage<LOGN, B0, 0>(x, tid, twg, twc, q);
  if constexpr (B0 > 0) {
    xchg_store<LOGN, B0>(buf, x, tid);
    if constexpr (warp_local<LOGN, B0 - 4>()) {
      __syncwarp();
    } else {
      __syncthreads();
    }
    xchg_load<LOGN, B0 - 4>(buf, x, tid);
    fwd_passes<LOGN, B0 - 4>(buf, x, tid, twg, twc, q);
  }
}

// LAZY: hand st() the unreduced outputs (< (2 LOGN + 1) q < 2^32 for 27-bit q),
// for consumers that accept any 32-bit operand (mont_mac).
template <int LOGN, bool LAZY = false, class LD, class ST>
__device__ __forceinline__ void ntt_fwd(NttState& ns, const uint2* __restrict__ twg, const uint2* twc,
                                        const Modulus& M, LD&& ld, ST&& st) {
  using C = NttCfg<LOGN>;
  const int tid = threadIdx.x;
  const u32 q = M.q;
  u32 x[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) x[r] = ld(tid | (r << C::SHIFT));
  u32* buf = ns.xbuf + ns.parity * C::N;
  ns.parity ^= 1;
  if constexpr (C::kFast) {
#ifndef EXP_NO_FWD
    fwd_passes<LOGN, LOGN - 4>(buf, x, tid, twg, twc, q);
#endif
    if constexpr (!LAZY) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {  // x < (2 LOGN + 1) q: Barrett to [0, 2q), then canonical
        const u32 v = x[r] - mulhi(x[r], M.barrett) * q;
        x[r] = csub(v, q);
      }
    }
    st(tid << 4, x);
  } else {
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[tid | (r << C::SHIFT)] = x[r];
    __syncthreads();
    for (int s = 0; s < LOGN; ++s) {
      const int t = C::N >> (s + 1);
      for (int b = tid; b < C::N / 2; b += C::T) {
        const int j = (b / t) * 2 * t + (b % t);
        const uint2 w = twg[(1 << s) + (j >> (LOGN - s))];
        const u32 u = buf[j];
        const u32 v = csub(mul_shoup(buf[j + t], w.x, w.y, q), q);
        buf[j] = mod_add(u, v, q);
        buf[j + t] = mod_sub(u, v, q);
      }
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = buf[(tid << 4) | r];
    st(tid << 4, x);
  }
}

// ---------------------------------------------------------------------------
// inverse

template <int LOGN, int B0>
__device__ __forceinline__ void inv_passes(u32* buf, u32 (&x)[16], int tid, const uint2* twg, const uint2* twc,
                                           u32 q) {
  inv_stage<LOGN, B0, 0>(x, tid, twg, twc, q);
  inv_stage<LOGN, B0, 1>(x, tid, twg, twc, q);
  inv_stage<LOGN, B0, 2>(x, tid, twg, twc, q);
  inv_stage<LOGN, B0, 3>(x, tid, twg, twc, q);
  if constexpr (B0 + 4 < LOGN) {
    xchg_store<LOGN, B0>(buf, x, tid);
    if constexpr (warp_local<LOGN, B0>()) {
      __syncwarp();
    } else {
      __syncthreads();
    }
    xchg_load<LOGN, B0 + 4>(buf, x, tid);
    inv_passes<LOGN, B0 + 4>(buf, x, tid, twg, twc, q);
  }
}

template <int LOGN, class LD16, class ST>
__device__ __forceinline__ void ntt_inv(NttState& ns, const uint2* __restrict__ twg, const uint2* twc,
                                        const Modulus& M, LD16&& ld16, ST&& st) {
  using C = NttCfg<LOGN>;
  const int tid = threadIdx.x;
  const u32 q = M.q;
  u32 x[16];
  u32* buf = ns.xbuf + ns.parity * C::N;
  ns.parity ^= 1;
  if constexpr (C::kFast) {
    ld16(tid << 4, x);
    inv_passes<LOGN, 0>(buf, x, tid, twg, twc, q);
#pragma unroll
    for (int r = 0; r < 16; ++r) st(tid | (r << C::SHIFT), r, csub(mul_shoup(x[r], M.ninv, M.ninv_sh, q), q));
  } else {
    ld16(tid << 4, x);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[(tid << 4) | r] = x[r];
    __syncthreads();
    for (int u = 0; u < LOGN; ++u) {
      const int t = 1 << u;
      for (int b = tid; b < C::N / 2; b += C::T) {
        const int j = (b / t) * 2 * t + (b % t);
        const uint2 w = twg[(1 << (LOGN - 1 - u)) + (j >> (u + 1))];
        const u32 a = buf[j], c = buf[j + t];
        buf[j] = mod_add(a, c, q);
        buf[j + t] = csub(mul_shoup(mod_sub(a, c, q), w.x, w.y, q), q);
      }
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int j = tid | (r << C::SHIFT);
      st(j, r, csub(mul_shoup(buf[j], M.ninv, M.ninv_sh, q), q));
    }
  }
}

}  // namespace gpir
