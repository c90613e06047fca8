// Client-side material on the GPU: the benchmark input factory.
//
// The reference generates every client's secret, expansion keys, RGSW(s) and
// queries on the CPU with numpy (src/he.py:220-271, 423-431, 487-515;
// src/protocol.py:246-281): ~0.6 s per client, minutes for the 256-512
// distinct clients of the large configs.  These kernels do the same
// arithmetic on the GPU from a counter-based hash RNG (so the samples differ
// from numpy's, the distributions and the encryption equations do not):
//   secret      s   ternary coefficients, NTT domain
//   error       e   centered binomial sum of `bound` coin-flip differences
//   encryption  (a, b) = (uniform in the NTT domain, phase - a s + NTT(e))
//   evk stage t rows i < ell: phase z^i tau_t(s), tau_t: X -> X^(n/2^t + 1)
//   RGSW(s)     rows i < ell: phase z^i s^2; rows ell + i: phase z^i s
//   query       phase NTT(payload): Delta / 2^stages at slot i*, and
//               z^dig / 2^stages at slot d0 + bit ell + dig for every set bit of j*
// All values are produced in the internal bit-reversed slot order and the
// keys go straight into the context's key pool (top-digit folded).
#pragma once
#include "kernels.cuh"

namespace gpir {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// independent streams: (seed, domain tag, row, index) -> 64 random bits
__device__ __forceinline__ uint64_t crng(uint64_t seed, uint32_t tag, uint32_t row, uint32_t idx) {
  return mix64(seed ^ mix64(((uint64_t)tag << 56) ^ ((uint64_t)row << 28) ^ idx));
}

// s: ternary coefficients (natural order) -> int8 copy + limbs mod q_i (natural)
__global__ void k_client_secret(uint64_t seed, int n, int K, int8_t* __restrict__ sc, u32* __restrict__ limbs,
                                Tables tb) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int v = (int)(crng(seed, 1, 0, j) % 3) - 1;
  sc[j] = (int8_t)v;
  for (int i = 0; i < K; ++i) limbs[(size_t)i * n + j] = v < 0 ? tb.mod[i].q - 1 : (u32)v;
}

// int8 coefficients -> limbs (natural order)
__global__ void k_client_lift(const int8_t* __restrict__ sc, int n, int K, u32* __restrict__ limbs, Tables tb) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int v = sc[j];
  for (int i = 0; i < K; ++i) limbs[(size_t)i * n + j] = v < 0 ? (u32)(tb.mod[i].q + v) : (u32)v;
}

// rows x K grid: out[row] = (a, phase[row] - a s + NTT(e_row)), all brv;
// s_brv (K, n); phase (rows, K, n) brv; errors regenerated per limb from the
// row's stream so every limb sees the same integer error polynomial.
template <int LOGN, int K>
__global__ void __launch_bounds__(NttCfg<LOGN>::T)
    k_client_encrypt(uint64_t seed, uint32_t row0, const u32* __restrict__ phase, const u32* __restrict__ s_brv,
                     u32* __restrict__ out, int bound, Tables tb, const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN;
  __shared__ __align__(16) u32 xbuf[2 * N];
  NttState ns{xbuf, 0};
  const int row = blockIdx.x, i = blockIdx.y;
  const Modulus M = tb.mod[i];
  const u32 q = M.q;
  const uint32_t r = row0 + row;
  u32* a_out = out + ((size_t)row * 2 * K + i) * N;
  u32* b_out = a_out + (size_t)K * N;
  const u32* ph = phase + ((size_t)row * K + i) * N;
  const u32* s = s_brv + (size_t)i * N;
  const uint64_t em = bound >= 32 ? ~0ull : ((1ull << bound) - 1);
  ntt_fwd<LOGN>(
      ns, tb.fwd + (size_t)i * N, tc.f[i], M,
      [&](int j) -> u32 {
        const uint64_t h = crng(seed, 2, r, j);
        const int e = __popcll(h & em) - __popcll((h >> 32) & em);
        return e < 0 ? (u32)((int)q + e) : (u32)e;
      },
      [&](int i0, const u32(&x)[16]) {
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
          const int slot = i0 + rr;
          const u32 a = (u32)(crng(seed, 3, r * 8 + i, slot) % q);
          a_out[slot] = a;
          b_out[slot] = mod_add(mod_sub(ph[slot], mod_mul(a, s[slot], M), q), x[rr], q);
        }
      });
}

// phases of the key rows (brv): evk rows (stages x ell) then RGSW rows (2 ell)
__global__ void k_client_key_phases(const u32* __restrict__ s_brv, int logn, int K, int stages, int ell,
                                    const u32* __restrict__ zpow /* [ell][K] */, u32* __restrict__ phase, Tables tb) {
  const int n = 1 << logn;
  const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t rows = (size_t)stages * ell + 2 * ell;
  if (g >= rows * K * n) return;
  const int slot = (int)(g % n), i = (int)((g / n) % K);
  const int row = (int)(g / ((size_t)K * n));
  const Modulus M = tb.mod[i];
  const u32* s = s_brv + (size_t)i * n;
  u32 base, zi;
  if (row < stages * ell) {
    const int t = row / ell;
    zi = zpow[(row % ell) * K + i];
    base = s[aut_src(slot, (u32)(n >> t) + 1, logn)];
  } else {
    const int rr = row - stages * ell;
    zi = zpow[(rr % ell) * K + i];
    const u32 sv = s[slot];
    base = rr < ell ? mod_mul(sv, sv, M) : sv;  // a-digit rows: z^i s^2; b-digit rows: z^i s
  }
  phase[g] = mod_mul(zi, base, M);
}

}  // namespace gpir
