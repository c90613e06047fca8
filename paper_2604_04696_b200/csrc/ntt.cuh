// Block-level negacyclic NTT / inverse NTT for one polynomial limb.
//
// One CTA of T = n/16 threads owns one n-point limb; every thread holds 16
// elements in registers.  The forward transform is Cooley-Tukey DIT with the
// psi twist merged into bit-reversed twiddles (natural coeffs -> brv evals);
// the inverse is Gentleman-Sande DIF (brv evals -> natural coeffs) with the
// n^{-1} scale applied at the end.  Both compute exactly the reference's
// transform (src/ring.py:408-453) up to the slot permutation documented in
// gpir_common.cuh.  Butterflies are Harvey-lazy with 32-bit Shoup products
// (values stay below 4q < 2^29 for 27-bit primes).
//
// For n = 2^LOGN with LOGN % 4 == 0 the transform runs as LOGN/4 radix-16
// passes over registers with shared-memory exchanges (xbuf, swizzled so all
// three access patterns are bank-conflict free at n = 4096); other sizes (the
// tiny test rings) use a simple shared-memory radix-2 loop with the same I/O
// contract.
//
// I/O contract (both paths):
//   forward: ld(j) is called for natural coefficient j = tid | r << (LOGN-4)
//            (r = 0..15);  st(i0, x[16]) receives brv slots i0 = 16*tid + r.
//   inverse: ld16(i0, x[16]) must fill brv slots i0 = 16*tid + r;
//            st(j, r, v) receives natural coefficient j = tid | r << (LOGN-4).
#pragma once
#include "gpir_common.cuh"

namespace gpir {

template <int LOGN>
struct NttCfg {
  static constexpr int N = 1 << LOGN;
  static constexpr int T = N / 16;
  static constexpr bool kFast = (LOGN % 4 == 0) && LOGN >= 8;
  static constexpr int SHIFT = LOGN - 4;
};

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

template <int LOGN, int B0>
__device__ __forceinline__ void fwd_pass(u32 (&x)[16], int tid, const uint2* __restrict__ tw, u32 q) {
  const u32 q2 = 2 * q;
#pragma unroll
  for (int rb = 3; rb >= 0; --rb) {
    const int s = LOGN - 1 - (B0 + rb);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & (1 << rb)) continue;
      const int j = pidx<B0>(tid, r);
      const uint2 w = __ldg(&tw[(1 << s) + (j >> (LOGN - s))]);
      const u32 u = csub(x[r], q2);
      const u32 t = mul_shoup(x[r | (1 << rb)], w.x, w.y, q);
      x[r] = u + t;
      x[r | (1 << rb)] = u + q2 - t;
    }
  }
}

template <int LOGN, int B0>
__device__ __forceinline__ void inv_pass(u32 (&x)[16], int tid, const uint2* __restrict__ tw, u32 q) {
  const u32 q2 = 2 * q;
#pragma unroll
  for (int rb = 0; rb < 4; ++rb) {
    const int u = B0 + rb;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r & (1 << rb)) continue;
      const int j = pidx<B0>(tid, r);
      const uint2 w = __ldg(&tw[(1 << (LOGN - 1 - u)) + (j >> (u + 1))]);
      const u32 a = x[r], b = x[r | (1 << rb)];
      x[r] = csub(a + b, q2);
      x[r | (1 << rb)] = mul_shoup(a + q2 - b, w.x, w.y, q);
    }
  }
}

template <int LOGN, int B0>
__device__ __forceinline__ void xchg_store(u32* xbuf, const u32 (&x)[16], int tid) {
#pragma unroll
  for (int r = 0; r < 16; ++r) xbuf[swz<LOGN>(pidx<B0>(tid, r))] = x[r];
}

template <int LOGN, int B0>
__device__ __forceinline__ void xchg_load(const u32* xbuf, u32 (&x)[16], int tid) {
#pragma unroll
  for (int r = 0; r < 16; ++r) x[r] = xbuf[swz<LOGN>(pidx<B0>(tid, r))];
}

// ---------------------------------------------------------------------------
// forward

template <int LOGN, int B0>
__device__ __forceinline__ void fwd_passes(u32* xbuf, u32 (&x)[16], int tid, const uint2* tw, u32 q) {
  fwd_pass<LOGN, B0>(x, tid, tw, q);
  if constexpr (B0 > 0) {
    __syncthreads();  // previous readers of xbuf are done
    xchg_store<LOGN, B0>(xbuf, x, tid);
    __syncthreads();
    xchg_load<LOGN, B0 - 4>(xbuf, x, tid);
    fwd_passes<LOGN, B0 - 4>(xbuf, x, tid, tw, q);
  }
}

template <int LOGN, class LD, class ST>
__device__ __forceinline__ void ntt_fwd(u32* xbuf, const uint2* __restrict__ tw, u32 q, LD&& ld, ST&& st) {
  using C = NttCfg<LOGN>;
  const int tid = threadIdx.x;
  u32 x[16];
  if constexpr (C::kFast) {
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = ld(tid | (r << C::SHIFT));
    fwd_passes<LOGN, LOGN - 4>(xbuf, x, tid, tw, q);
    const u32 q2 = 2 * q;
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = csub(csub(x[r], q2), q);
    st(tid << 4, x);
  } else {
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = ld(tid | (r << C::SHIFT));
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) xbuf[tid | (r << C::SHIFT)] = x[r];
    __syncthreads();
    for (int s = 0; s < LOGN; ++s) {
      const int t = C::N >> (s + 1);
      for (int b = tid; b < C::N / 2; b += C::T) {
        const int j = (b / t) * 2 * t + (b % t);
        const uint2 w = tw[(1 << s) + (j >> (LOGN - s))];
        const u32 u = xbuf[j];
        const u32 v = csub(mul_shoup(xbuf[j + t], w.x, w.y, q), q);
        xbuf[j] = mod_add(u, v, q);
        xbuf[j + t] = mod_sub(u, v, q);
      }
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = xbuf[(tid << 4) | r];
    st(tid << 4, x);
  }
}

// ---------------------------------------------------------------------------
// inverse

template <int LOGN, int B0>
__device__ __forceinline__ void inv_passes(u32* xbuf, u32 (&x)[16], int tid, const uint2* tw, u32 q) {
  inv_pass<LOGN, B0>(x, tid, tw, q);
  if constexpr (B0 + 4 < LOGN) {
    __syncthreads();
    xchg_store<LOGN, B0>(xbuf, x, tid);
    __syncthreads();
    xchg_load<LOGN, B0 + 4>(xbuf, x, tid);
    inv_passes<LOGN, B0 + 4>(xbuf, x, tid, tw, q);
  }
}

template <int LOGN, class LD16, class ST>
__device__ __forceinline__ void ntt_inv(u32* xbuf, const uint2* __restrict__ tw, const Modulus& M, LD16&& ld16,
                                        ST&& st) {
  using C = NttCfg<LOGN>;
  const int tid = threadIdx.x;
  const u32 q = M.q;
  u32 x[16];
  if constexpr (C::kFast) {
    ld16(tid << 4, x);
    inv_passes<LOGN, 0>(xbuf, x, tid, tw, q);
#pragma unroll
    for (int r = 0; r < 16; ++r) st(tid | (r << C::SHIFT), r, csub(mul_shoup(x[r], M.ninv, M.ninv_sh, q), q));
  } else {
    ld16(tid << 4, x);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) xbuf[(tid << 4) | r] = x[r];
    __syncthreads();
    for (int u = 0; u < LOGN; ++u) {
      const int t = 1 << u;
      for (int b = tid; b < C::N / 2; b += C::T) {
        const int j = (b / t) * 2 * t + (b % t);
        const uint2 w = tw[(1 << (LOGN - 1 - u)) + (j >> (u + 1))];
        const u32 a = xbuf[j], c = xbuf[j + t];
        xbuf[j] = mod_add(a, c, q);
        xbuf[j + t] = csub(mul_shoup(mod_sub(a, c, q), w.x, w.y, q), q);
      }
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int j = tid | (r << C::SHIFT);
      st(j, r, csub(mul_shoup(xbuf[j], M.ninv, M.ninv_sh, q), q));
    }
  }
}

}  // namespace gpir
