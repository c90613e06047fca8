// libgpir: host engine + C ABI (include/gpir.h) for the GPIR server pipeline
// on B200 (sm_100a).  One context per device; all device memory is owned by
// the context (keys, DB, pooled per-batch workspace); work is issued on one
// stream per call and timed with CUDA events per phase.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <atomic>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/gpir.h"
#include "kernels.cuh"
#include "rowsel_tc.cuh"
#include "stage_kernels.cuh"
#include "client.cuh"

// hybrid planner thresholds (nodes / ciphertexts per stage, whole batch)
// ExpandQuery: with the node-batched MAC (k_op_eq_mac_nb) the operation-level
// executor is faster than the stage kernel at every stage size (r1g: eq8 2.73
// vs 3.02 ms at config 2, ExpandQuery 22.7 vs 25.2 ms at config 3), so the
// stage-level threshold is out of reach; mode 3 stays selectable per stage.
static constexpr size_t kEqStageNodes = (size_t)1 << 62;
static constexpr size_t kXpStageCts = 64;  // r1g: ColTor levels of 64-128 pairs are faster stage-level

using namespace gpir;

static thread_local std::string g_err;

#define FAIL(code, msg)  \
  do {                   \
    g_err = (msg);       \
    return (code);       \
  } while (0)

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e_);                       \
      return GPIR_CUDA_ERROR;                                                           \
    }                                                                                   \
  } while (0)

// kernels launched eagerly by this library (graph replays not included): gpir_launch_count
static std::atomic<uint64_t> g_launches{0};

#define CKL()                                                                            \
  do {                                                                                   \
    g_launches.fetch_add(1, std::memory_order_relaxed);                                  \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess) {                                                             \
      g_err = std::string("kernel launch (gpir.cu:") + std::to_string(__LINE__) + "): " + cudaGetErrorString(e_); \
      return GPIR_CUDA_ERROR;                                                            \
    }                                                                                    \
  } while (0)

typedef unsigned __int128 u128;

// ---------------------------------------------------------------------------
// device buffer helper

// bumped by every (re)allocation of a device buffer: captured CUDA graphs
// hold raw pointers, so a graph is only replayed while this is unchanged
static std::atomic<uint64_t> g_alloc_gen{0};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t want) {
    if (want <= bytes) return 0;
    ++g_alloc_gen;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (want == 0) return 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      g_err = std::string("cudaMalloc(") + std::to_string(want) + "): " + cudaGetErrorString(e);
      p = nullptr;
      return GPIR_CUDA_ERROR;
    }
    bytes = want;
    return 0;
  }
  void release() {
    if (p) {
      cudaFree(p);
      ++g_alloc_gen;
    }
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

struct gpir_db {
  uint32_t d0 = 0, d1 = 0;
  DevBuf data;  // (d1, d0, k, n) brv
  DevBuf d8;    // tensor-core byte planes D8[p][c][ntile][plane][g][NT][16], packed on first use
  int d8_nt = 0, d8_kc = 0;
  // capacity mode (gpir_db_compact): only the byte planes in the k_rowsel_tk
  // layout are kept; the u32 copy is released (the DB then occupies its encoded
  // size once in HBM) and every batch runs the TMEM-resident RowSel
  bool compact = false;
};

struct gpir_ctx {
  int device = 0;
  uint32_t n = 0, logn = 0, k = 0, ell = 0, z_bits = 0;
  std::vector<uint32_t> q, psi;
  Tables tb{};
  CrtConst cc{};
  TwConst tc{};
  FoldConst fc{};
  int stage_timing = 0;
  size_t sel_budget = 0;  // capacity path: bytes of the (B, window) RowSel selection (0: env / 16 GiB)
  int max_batch = 0;      // capacity path: largest sub-batch (0: from the free device memory)
  // per-phase device time of a batch with stats: intervals between pooled events,
  // summed over column windows and sub-batches (phase: 0 EQ, 1 RGSW, 2 pack, 3 GEMM,
  // 4 transpose, 5 ColTor)
  std::vector<cudaEvent_t> evp;
  size_t evp_used = 0;
  struct Interval {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<Interval> plog;
  cudaEvent_t ev_next() {
    if (evp_used == evp.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      evp.push_back(e);
    }
    return evp[evp_used++];
  }
  struct SubBatch {
    const gpir_db* db;
    int B;
    uint64_t gen;
    int bs;
  };
  std::vector<SubBatch> subbatch_cache;
  uint32_t error_bound = 16;
  std::vector<gpir_stage_time> last_stages;
  DevBuf tw_fwd, tw_inv, mono;
  // key pool
  uint32_t key_slots = 0, key_stages = 0;
  std::vector<int> slot_stages;  // -1 = empty
  std::vector<char> slot_rgsw;
  DevBuf evk_pool, rgsw_pool;
  // workspace
  DevBuf ws_state0, ws_state1, ws_arows, ws_sel, ws_ct0, ws_ct1, ws_kslot, ws_crows, ws_y, ws_part;
  DevBuf ws_coeff, ws_dig, ws_dn, ws_io0, ws_io1, ws_a8;
  int rowsel_engine = 0;  // 0 auto, 1 CUDA cores, 2 tensor cores
  int num_sms = 148;
  // row-sharded session state (gpir_sharded_expand -> gpir_sharded_coltor)
  u32* sh_leaves = nullptr;
  uint32_t sh_B = 0, sh_d0 = 0, sh_d1 = 0, sh_total = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[13];
  cudaEvent_t ev_legacy = nullptr;  // orders the private stream after the legacy default stream (pick_stream)
  // CUDA graphs of the device pipeline (answer_dev), keyed by everything the
  // captured launches bake in; the first call of a key runs eagerly (lazy
  // allocations, DB byte-plane packing), the second captures, later ones replay
  struct GraphEntry {
    const void* db = nullptr;
    const void* dq = nullptr;
    const void* dout = nullptr;
    int B = 0;
    uint64_t gen = 0;
    std::vector<uint8_t> modes;
    int state = 0;  // 1 seen once, 2 captured, -1 capture failed (stay eager)
    cudaGraphExec_t exec = nullptr;
  };
  std::vector<GraphEntry> graphs;
  int use_graph = 1;  // GPIR_GRAPH=0 disables
  std::mutex mu;
  size_t ct_words() const { return 2 * (size_t)k * n; }
};

// ---------------------------------------------------------------------------
// host-side math for tables

static uint64_t powmod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = (u128)r * b % m;
    b = (u128)b * b % m;
    e >>= 1;
  }
  return r;
}
static uint32_t shoup(uint32_t w, uint32_t q) { return (uint32_t)(((uint64_t)w << 32) / q); }
static uint32_t hbrv(uint32_t x, int logn) {
  uint32_t r = 0;
  for (int b = 0; b < logn; ++b) r |= ((x >> b) & 1u) << (logn - 1 - b);
  return r;
}

static int build_tables(gpir_ctx* c) {
  const uint32_t n = c->n, k = c->k;
  std::vector<uint2> fwd((size_t)k * n), inv((size_t)k * n), mono((size_t)c->logn * k * n);
  for (uint32_t i = 0; i < k; ++i) {
    const uint32_t q = c->q[i];
    const uint64_t psi = c->psi[i];
    const uint64_t ipsi = powmod(psi, q - 2, q);
    std::vector<uint32_t> pw(2 * n), ipw(2 * n);
    uint64_t v = 1, iv = 1;
    for (uint32_t e = 0; e < 2 * n; ++e) {
      pw[e] = (uint32_t)v;
      ipw[e] = (uint32_t)iv;
      v = v * psi % q;
      iv = iv * ipsi % q;
    }
    for (uint32_t m = 0; m < n; ++m) {
      const uint32_t w = pw[hbrv(m, c->logn)], iw = ipw[hbrv(m, c->logn)];
      fwd[(size_t)i * n + m] = make_uint2(w, shoup(w, q));
      inv[(size_t)i * n + m] = make_uint2(iw, shoup(iw, q));
      if (i < (uint32_t)kTwConstLimbs && m < (uint32_t)kTwConstEntries) {
        c->tc.f[i][m] = fwd[(size_t)i * n + m];
        c->tc.i[i][m] = inv[(size_t)i * n + m];
      }
    }
    // X^{-2^t} in brv layout: slot s holds psi^((2 brv(s) + 1) e), e = -2^t mod 2n  (src/ring.py:667-673)
    for (uint32_t t = 0; t < c->logn; ++t) {
      const uint64_t e = (2ull * n - (1ull << t)) % (2ull * n);
      for (uint32_t s = 0; s < n; ++s) {
        const uint64_t ex = ((2ull * hbrv(s, c->logn) + 1) * e) % (2ull * n);
        const uint32_t w = pw[ex];
        mono[((size_t)t * k + i) * n + s] = make_uint2(w, shoup(w, q));
      }
    }
    Modulus& M = c->tb.mod[i];
    M.q = q;
    uint32_t inv32 = 1;  // q^{-1} mod 2^32 by Newton
    for (int it = 0; it < 5; ++it) inv32 *= 2 - q * inv32;
    M.qinv_neg = (uint32_t)(0u - inv32);
    M.r2 = (uint32_t)((((u128)1) << 64) % q);
    M.r1 = (uint32_t)((1ull << 32) % q);
    M.r1_sh = shoup(M.r1, q);
    M.barrett = (uint32_t)((1ull << 32) / q);
    M.ninv = (uint32_t)powmod(n, q - 2, q);
    M.ninv_sh = shoup(M.ninv, q);
  }
  // CRT constants (src/ring.py:214-235)
  u128 Q = 1;
  for (uint32_t i = 0; i < k; ++i) Q *= c->q[i];
  CrtConst& cc = c->cc;
  cc.k = (int)k;
  cc.ell = (int)c->ell;
  cc.z_bits = (int)c->z_bits;
  cc.logn = (int)c->logn;
  for (uint32_t i = 0; i < k; ++i) {
    const u128 m = Q / c->q[i];
    cc.m_lo[i] = (uint64_t)m;
    cc.m_hi[i] = (uint64_t)(m >> 64);
    const uint32_t mh = (uint32_t)powmod((uint64_t)(m % c->q[i]), c->q[i] - 2, c->q[i]);
    c->tb.mod[i].mhat = mh;
    c->tb.mod[i].mhat_sh = shoup(mh, c->q[i]);
  }
  cc.q_lo = (uint64_t)Q;
  cc.q_hi = (uint64_t)(Q >> 64);
  const u128 half = (Q - 1) / 2;
  cc.half_lo = (uint64_t)half;
  cc.half_hi = (uint64_t)(half >> 64);
  uint32_t t = 1;
  while (t < k) t *= 2;
  cc.n_red = 0;
  while (t >= 1) {
    const u128 r = Q * t;
    cc.red_lo[cc.n_red] = (uint64_t)r;
    cc.red_hi[cc.n_red] = (uint64_t)(r >> 64);
    ++cc.n_red;
    t /= 2;
  }
  u128 dc = 0;
  for (uint32_t j = 0; j + 1 < c->ell; ++j) dc += (((u128)1 << (c->z_bits - 1)) - 1) << (c->z_bits * j);
  cc.dc_lo = (uint64_t)dc;
  cc.dc_hi = (uint64_t)(dc >> 64);
  // top-digit fold constants (k_fold_rows): z^(j-(ell-1)) and z^-(ell-1) mod q_i
  for (uint32_t i = 0; i < k; ++i) {
    const uint64_t qi = c->q[i];
    const uint64_t zinv = powmod(powmod(2, c->z_bits, qi), qi - 2, qi);
    for (uint32_t j = 0; j < c->ell; ++j) {
      const uint32_t e = (j + 1 < c->ell) ? c->ell - 1 - j : c->ell - 1;
      const uint32_t w = (uint32_t)powmod(zinv, e, qi);
      c->fc.w[i][j] = make_uint2(w, shoup(w, (uint32_t)qi));
    }
  }
  int rc;
  if ((rc = c->tw_fwd.ensure(fwd.size() * sizeof(uint2)))) return rc;
  if ((rc = c->tw_inv.ensure(inv.size() * sizeof(uint2)))) return rc;
  if ((rc = c->mono.ensure(mono.size() * sizeof(uint2)))) return rc;
  CK(cudaMemcpy(c->tw_fwd.p, fwd.data(), fwd.size() * sizeof(uint2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->tw_inv.p, inv.data(), inv.size() * sizeof(uint2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->mono.p, mono.data(), mono.size() * sizeof(uint2), cudaMemcpyHostToDevice));
  c->tb.fwd = c->tw_fwd.as<uint2>();
  c->tb.inv = c->tw_inv.as<uint2>();
  return 0;
}

// ---------------------------------------------------------------------------
// geometry (src/planner.py:153-173)

// The stream a device-pointer entry point runs on: the caller's, or (NULL) the
// context's private stream ordered after all work already queued on the legacy
// default stream -- e.g. a collective or copy torch issued on stream 0 -- so
// NULL behaves like the default stream for the caller (the call then also
// synchronises before returning).
static cudaStream_t pick_stream(gpir_ctx* c, void* stream) {
  if (stream) return (cudaStream_t)stream;
  if (cudaEventRecord(c->ev_legacy, cudaStreamLegacy) == cudaSuccess) cudaStreamWaitEvent(c->stream, c->ev_legacy, 0);
  return c->stream;
}

static uint32_t ilog2(uint32_t v) {
  uint32_t r = 0;
  while ((1u << r) < v) ++r;
  return r;
}
static uint32_t leaves_of(uint32_t d0, uint32_t d1, uint32_t ell) { return d0 + ilog2(d1) * ell; }
static uint32_t stages_of(uint32_t total) { return total > 1 ? ilog2(total) : 0; }

// ---------------------------------------------------------------------------
// templated engine

static int bitrev_rows(gpir_ctx* c, const uint32_t* in, uint32_t* out, size_t rows, cudaStream_t s) {
  const size_t tot = rows << c->logn;
  if (!tot) return 0;
  k_bitrev_rows<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(in, out, rows, (int)c->logn);
  CKL();
  return 0;
}

// Top-digit fold (k_fold_rows) of B x G row groups of ell rows each: group
// (b, g) at src + b*sb + g*sg -> dst + b*db + g*dg (words; may alias).
static int fold_rows(gpir_ctx* c, const uint32_t* src, uint32_t* dst, int B, int G, size_t sb, size_t sg, size_t db,
                     size_t dg, cudaStream_t s) {
  const size_t tot = (size_t)B * G * (2 * (size_t)c->k << c->logn);
  if (!tot) return 0;
  const unsigned grid = (unsigned)((tot + 255) / 256);
  switch (c->ell) {
    case 5:
      k_fold_rows<5><<<grid, 256, 0, s>>>(src, dst, B, G, sb, sg, db, dg, (int)c->logn, (int)c->k, c->tb, c->fc);
      break;
    case 6:
      k_fold_rows<6><<<grid, 256, 0, s>>>(src, dst, B, G, sb, sg, db, dg, (int)c->logn, (int)c->k, c->tb, c->fc);
      break;
    default:
      FAIL(GPIR_UNSUPPORTED, "fold: unsupported ell");
  }
  CKL();
  return 0;
}

// Per-stage device timing for plan tuning (GPIR_STAGE_PROF=1): events on the
// launch stream, printed to stderr at the end of each batch.
struct StageProf {
  bool env = getenv("GPIR_STAGE_PROF") != nullptr;
  bool fine = env && atoi(getenv("GPIR_STAGE_PROF")) >= 2;  // also between the kernels of a stage
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<std::string> lab;
  std::vector<gpir_stage_time> info;
  size_t n = 0;
  void begin(bool ctx_on) {
    on = env || ctx_on;
    n = 0;
  }
  void mark(cudaStream_t s, const std::string& l, int phase = -1, int stage = 0, int mode = 0, uint32_t units = 0) {
    if (!on) return;
    if (n == ev.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
      lab.emplace_back();
      info.emplace_back();
    }
    lab[n] = l;
    info[n] = gpir_stage_time{(uint8_t)(phase < 0 ? 255 : phase), (uint8_t)mode, (uint16_t)stage, units, 0.f};
    cudaEventRecord(ev[n++], s);
  }
  // per-interval times; phase entries (phase != 255) are returned, labels printed under GPIR_STAGE_PROF
  void flush(std::vector<gpir_stage_time>* out) {
    if (!on || n < 2) return;
    cudaEventSynchronize(ev[n - 1]);
    if (out) out->clear();
    float acc = 0;
    for (size_t i = 1; i < n; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      if (env) fprintf(stderr, "[stage prof] %-16s %8.3f ms\n", lab[i].c_str(), ms);
      acc += ms;
      if (info[i].phase != 255) {  // fine-grained sub-marks fold into the next stage entry
        if (out) {
          gpir_stage_time t = info[i];
          t.ms = acc;
          out->push_back(t);
        }
        acc = 0;
      }
    }
    n = 0;
    on = false;
    cudaGetLastError();
  }
};
static thread_local StageProf g_sprof;

// Dynamic shared memory attribute of a kernel, per device, only ever raised:
// the kernels are shared by every Engine instantiation, so one global record
// (a per-instantiation cache could lower the attribute below what another
// instantiation's launch needs, failing it with "invalid argument").  Set
// outside graph captures (the first, eager call of a shape).
static int raise_smem_attr(int device, const void* kern, size_t smem) {
  static std::mutex mu;
  static std::vector<std::tuple<int, const void*, size_t>> smem_set;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& ks : smem_set)
    if (std::get<0>(ks) == device && std::get<1>(ks) == kern) {
      if (std::get<2>(ks) >= smem) return 0;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      std::get<2>(ks) = smem;
      return 0;
    }
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  smem_set.emplace_back(device, kern, smem);
  return 0;
}

template <int LOGN, int K, int ELL>
struct Engine {
  static constexpr int N = 1 << LOGN;
  static constexpr int T = NttCfg<LOGN>::T;
  static constexpr size_t CT = 2 * (size_t)K * N;
  static size_t fused_smem() {
    return (size_t)NttCfg<LOGN>::XBUF_WORDS * 4 + (size_t)priv_slots<K, ELL>() * 16 * T * 4 + 16;  // + mbarrier
  }

  static int setup_attrs() {
    static bool done = false;
    if (done) return 0;
    const int sm = (int)fused_smem();
    CK(cudaFuncSetAttribute(k_eq_fused<LOGN, K, ELL>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute(k_xp_fused<LOGN, K, ELL>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute(k_eq_nttmac<LOGN, K, ELL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)k2eq_dyn_smem<LOGN>()));
    done = true;
    return 0;
  }

  // op-level scratch sizing: nodes per chunk bounded by ~1 GiB
  static size_t op_chunk(size_t per_node_words) {
    static const double genv = getenv("GPIR_OP_BUDGET_GIB") ? atof(getenv("GPIR_OP_BUDGET_GIB")) : 2.0;
    const size_t budget = (size_t)(genv * (double)(1ull << 28));  // words (default 2 GiB): a config-2 stage per chunk
    return std::max<size_t>(1, budget / per_node_words);
  }

  // one ExpandQuery stage: state (B, C) -> out (B, Cout)
  // a8f (operation-level mode only): write the row leaves (outputs c < d0) as
  // RowSel byte planes in that layout instead of u32 words (k_op_eq_mac_a8q)
  static int expand_stage(gpir_ctx* c, const u32* state, int B, int C, u32* out, int Cout, int t, RowsDesc ksk,
                          int mode, cudaStream_t s, uint32_t* launches, const A8Desc* a8f = nullptr, int d0 = 0) {
    const u32 k_aut = (u32)(N >> t) + 1;
    const uint2* mono = c->mono.as<uint2>() + (size_t)t * K * N;
    int rc;
    if (mode == 1) {  // stage-fused: one CTA per node (all limbs and digits resident in shared memory)
      if ((rc = setup_attrs())) return rc;
      k_eq_fused<LOGN, K, ELL><<<B * C, T, fused_smem(), s>>>(state, C, out, Cout, ksk, k_aut, mono, c->tb, c->cc, c->tc);
      CKL();
      ++*launches;
      return 0;
    }
    if (mode == 2) {  // split stage-fused: K1 (iNTT + Dcp per node) -> K2 (digit NTT + MAC + combine per node x limb)
      if ((rc = setup_attrs())) return rc;
      const size_t nodes = (size_t)B * C;
      const size_t cn = std::min(nodes, op_chunk((size_t)ELL * N));
      if ((rc = c->ws_dig.ensure(cn * ELL * N * 4))) return rc;
      for (size_t n0 = 0; n0 < nodes; n0 += cn) {
        const int nn = (int)std::min(cn, nodes - n0);
        k_eq_dcp<LOGN, K, ELL><<<nn, T, 0, s>>>(state, (int)n0, k_aut, c->ws_dig.as<int>(), c->tb, c->cc, c->tc);
        CKL();
        k_eq_nttmac<LOGN, K, ELL><<<nn * K, T, k2eq_dyn_smem<LOGN>(), s>>>(
            state, C, (int)n0, c->ws_dig.as<int>(), ksk, k_aut, mono, out, Cout, c->tb, c->tc);
        CKL();
        *launches += 2;
      }
      return 0;
    }
    const size_t per = (size_t)K * N + (size_t)ELL * N + (mode == 3 ? 0 : (size_t)ELL * K * N);
    static const size_t chunk_env = getenv("GPIR_OP_CHUNK") ? (size_t)atol(getenv("GPIR_OP_CHUNK")) : 0;
    size_t chunk = chunk_env ? chunk_env : op_chunk(per);
    if (chunk >= 16) chunk &= ~(size_t)15;  // node groups of the batched MACs never straddle a chunk
    if (a8f) chunk = std::max<size_t>(1, chunk / C) * C;  // the fused last stage: whole queries per chunk
    const size_t nodes = (size_t)B * C;
    const size_t cn = std::min(chunk, nodes);
    if ((rc = c->ws_coeff.ensure(cn * K * N * 4))) return rc;
    if ((rc = c->ws_dig.ensure(cn * ELL * N * 4))) return rc;
    if (mode != 3 && (rc = c->ws_dn.ensure(cn * ELL * K * N * 4))) return rc;
    if (mode == 3 && (rc = setup_attrs())) return rc;
    for (size_t n0 = 0; n0 < nodes; n0 += cn) {
      const int nn = (int)std::min(cn, nodes - n0);
      k_op_eq_intt<LOGN, K><<<dim3(nn, K), T, 0, s>>>(state, (int)n0, k_aut, c->ws_coeff.as<u32>(), c->tb, c->tc);
      CKL();
      if (g_sprof.fine) g_sprof.mark(s, "  eq_intt");
      const size_t tot = (size_t)nn * N;
      k_op_dcp<LOGN, K, ELL><<<(unsigned)((tot / 4 + 255) / 256), 256, 0, s>>>(c->ws_coeff.as<u32>(), nn,
                                                                          c->ws_dig.as<int>(), c->tb, c->cc, ELL - 1);
      CKL();
      if (g_sprof.fine) g_sprof.mark(s, "  eq_dcp");
      if (mode == 3) {  // hybrid: the digit NTTs stream straight into the key-switch MAC (K2)
        k_eq_nttmac<LOGN, K, ELL><<<nn * K, T, k2eq_dyn_smem<LOGN>(), s>>>(state, C, (int)n0, c->ws_dig.as<int>(), ksk, k_aut, mono,
                                                       out, Cout, c->tb, c->tc);
        CKL();
        *launches += 3;
        continue;
      }
      k_op_digit_ntt<LOGN, K, ELL><<<dim3(nn * (ELL - 1), K), T, 0, s>>>(c->ws_dig.as<int>(), c->ws_dn.as<u32>(), c->tb,
                                                                        c->tc);
      CKL();
      if (g_sprof.fine) g_sprof.mark(s, "  eq_dntt");
      static const int mac_nb = getenv("GPIR_MAC_NB") ? atoi(getenv("GPIR_MAC_NB")) : 108;
      if (a8f) {  // last stage: row leaves straight into the RowSel A operand (+ the other nodes as usual)
        const int b0 = (int)(n0 / C), nq = nn / C;
        dim3 g((N / 8) * K, (nq + 31) / 32, d0 / 16);
        k_op_eq_mac_a8q<LOGN, K, ELL><<<g, 256, 0, s>>>(state, C, b0, nq, c->ws_dn.as<u32>(), ksk, k_aut, mono, out,
                                                        Cout, c->tb, *a8f);
        if (d0 < C) {
          CKL();
          const size_t tm = ((size_t)(nn + 7) / 8) * K * (N / 4);
          k_op_eq_mac_nb4<LOGN, K, ELL, 8><<<(unsigned)((tm + 255) / 256), 256, 0, s>>>(
              state, C, (int)n0, nn, c->ws_dn.as<u32>(), ksk, k_aut, mono, out, Cout, c->tb, d0);
          ++*launches;
        }
      } else if (mac_nb == 4 || mac_nb == 104 || mac_nb == 108 || mac_nb == 116) {  // 4 slots per thread, NB nodes
        const int nb = mac_nb == 4 ? 4 : mac_nb - 100;
        const size_t tm = ((size_t)(nn + nb - 1) / nb) * K * (N / 4);
        auto kern = nb == 4 ? k_op_eq_mac_nb4<LOGN, K, ELL, 4>
                    : nb == 8 ? k_op_eq_mac_nb4<LOGN, K, ELL, 8> : k_op_eq_mac_nb4<LOGN, K, ELL, 16>;
        kern<<<(unsigned)((tm + 255) / 256), 256, 0, s>>>(state, C, (int)n0, nn, c->ws_dn.as<u32>(), ksk, k_aut,
                                                           mono, out, Cout, c->tb, 0);
      } else if (mac_nb == 8 || mac_nb == 16 || mac_nb == 32) {  // NB nodes per thread: key rows loaded once per group
        const size_t tm = ((size_t)(nn + mac_nb - 1) / mac_nb) * K * N;
        auto kern = mac_nb == 8 ? k_op_eq_mac_nb<LOGN, K, ELL, 8>
                    : mac_nb == 16 ? k_op_eq_mac_nb<LOGN, K, ELL, 16> : k_op_eq_mac_nb<LOGN, K, ELL, 32>;
        kern<<<(unsigned)((tm + 255) / 256), 256, 0, s>>>(state, C, (int)n0, nn, c->ws_dn.as<u32>(), ksk, k_aut,
                                                           mono, out, Cout, c->tb);
      } else {
        const size_t tm = (size_t)nn * K * N;
        k_op_eq_mac<LOGN, K, ELL><<<(unsigned)((tm + 255) / 256), 256, 0, s>>>(
            state, C, (int)n0, nn, c->ws_dn.as<u32>(), ksk, k_aut, mono, out, Cout, c->tb);
      }
      CKL();
      if (g_sprof.fine) g_sprof.mark(s, "  eq_mac");
      *launches += 4;
    }
    return 0;
  }

  // batched external products: (B, M) cts (or ColTor pairs) -> out (B, M)
  static int ext_product(gpir_ctx* c, const u32* in, size_t in_b, int B, int M, int pairs, u32* out, size_t out_b,
                         RowsDesc rows, int mode, cudaStream_t s, uint32_t* launches) {
    int rc;
    if (B * M == 0) return 0;
    if (mode == 1) {
      if ((rc = setup_attrs())) return rc;
      k_xp_fused<LOGN, K, ELL><<<B * M, T, fused_smem(), s>>>(in, in_b, M, pairs, out, out_b, rows, c->tb, c->cc, c->tc);
      CKL();
      ++*launches;
      return 0;
    }
    if (mode == 2) {
      if ((rc = setup_attrs())) return rc;
      const size_t cts = (size_t)B * M;
      const size_t cn = std::min(cts, op_chunk((size_t)2 * ELL * N));
      if ((rc = c->ws_dig.ensure(cn * 2 * ELL * N * 4))) return rc;
      for (size_t m0 = 0; m0 < cts; m0 += cn) {
        const int nn = (int)std::min(cn, cts - m0);
        k_xp_dcp<LOGN, K, ELL><<<nn, T, 0, s>>>(in, in_b, M, (int)m0, pairs, c->ws_dig.as<int>(), c->tb, c->cc, c->tc);
        CKL();
        launch_xp_nttmac<LOGN, K, ELL>(nn * K, s, in, in_b, M, (int)m0, pairs, c->ws_dig.as<int>(), rows, out, out_b,
                                       c->tb, c->tc);
        CKL();
        *launches += 2;
      }
      return 0;
    }
    const size_t per = 2 * ((size_t)K * N + (size_t)ELL * N + (mode == 3 ? 0 : (size_t)ELL * K * N));
    const size_t chunk = op_chunk(per);
    const size_t cts = (size_t)B * M;
    const size_t cn = std::min(chunk, cts);
    if ((rc = c->ws_coeff.ensure(cn * 2 * K * N * 4))) return rc;
    if ((rc = c->ws_dig.ensure(cn * 2 * ELL * N * 4))) return rc;
    if (mode != 3 && (rc = c->ws_dn.ensure(cn * 2 * ELL * K * N * 4))) return rc;
    if (mode == 3 && (rc = setup_attrs())) return rc;
    for (size_t m0 = 0; m0 < cts; m0 += cn) {
      const int nn = (int)std::min(cn, cts - m0);
      k_op_xp_intt<LOGN, K><<<dim3(2 * nn, K), T, 0, s>>>(in, in_b, M, (int)m0, pairs, c->ws_coeff.as<u32>(), c->tb, c->tc);
      CKL();
      if (g_sprof.fine) g_sprof.mark(s, "  xp_intt");
      const size_t tot = (size_t)2 * nn * N;
      k_op_dcp<LOGN, K, ELL><<<(unsigned)((tot / 4 + 255) / 256), 256, 0, s>>>(c->ws_coeff.as<u32>(), 2 * nn,
                                                                          c->ws_dig.as<int>(), c->tb, c->cc, ELL - 1);
      CKL();
      if (g_sprof.fine) g_sprof.mark(s, "  xp_dcp");
      if (mode == 3) {
        launch_xp_nttmac<LOGN, K, ELL>(nn * K, s, in, in_b, M, (int)m0, pairs, c->ws_dig.as<int>(), rows, out, out_b,
                                       c->tb, c->tc);
        CKL();
        if (g_sprof.fine) g_sprof.mark(s, "  xp_nttmac");
        *launches += 3;
        continue;
      }
      k_op_digit_ntt<LOGN, K, ELL><<<dim3(2 * nn * (ELL - 1), K), T, 0, s>>>(c->ws_dig.as<int>(), c->ws_dn.as<u32>(),
                                                                            c->tb, c->tc);
      CKL();
      // 8 cts per thread, one slot each: the 4-slot variant needs 2 x 4 ELL key registers (130 in all) and
      // loses more to occupancy than it saves in load instructions (ColTor level 0: 0.884 vs 0.798 ms)
      static const int xmac_nb = getenv("GPIR_XMAC_NB") ? atoi(getenv("GPIR_XMAC_NB")) : 8;
      if (xmac_nb == 104 || xmac_nb == 108) {  // 4 slots per thread (128-bit accesses), NB cts
        const int nb = xmac_nb - 100;
        const size_t tm = ((size_t)(nn + nb - 1) / nb) * K * (N / 4);
        auto kern = nb == 4 ? k_op_xp_mac_nb4<LOGN, K, ELL, 4> : k_op_xp_mac_nb4<LOGN, K, ELL, 8>;
        kern<<<(unsigned)((tm + 255) / 256), 256, 0, s>>>(in, in_b, M, (int)m0, nn, pairs, c->ws_dn.as<u32>(), rows,
                                                           out, out_b, c->tb);
      } else if (xmac_nb == 8 || xmac_nb == 16) {  // NB cts per thread: key rows loaded once per group
        const size_t tm = ((size_t)(nn + xmac_nb - 1) / xmac_nb) * K * N;
        auto kern = xmac_nb == 8 ? k_op_xp_mac_nb<LOGN, K, ELL, 8> : k_op_xp_mac_nb<LOGN, K, ELL, 16>;
        kern<<<(unsigned)((tm + 255) / 256), 256, 0, s>>>(in, in_b, M, (int)m0, nn, pairs, c->ws_dn.as<u32>(), rows,
                                                           out, out_b, c->tb);
      } else {
        const size_t tm = (size_t)nn * K * N;
        k_op_xp_mac<LOGN, K, ELL><<<(unsigned)((tm + 255) / 256), 256, 0, s>>>(in, in_b, M, (int)m0, nn, pairs,
                                                                               c->ws_dn.as<u32>(), rows, out, out_b,
                                                                               c->tb);
      }
      CKL();
      *launches += 4;
    }
    return 0;
  }

  static bool tc_eligible(gpir_ctx* c, int B, const gpir_db* db) {
    const int KN = K * N;
    if (c->rowsel_engine == 1) return false;
    return db->d0 <= 1024 && KN % PK_P == 0;
  }

  // byte-plane packing of R rows x Kd into the canonical tiles (k_pack_planes2
  // with 32 p per CTA; GPIR_PACK=16: 16 p, GPIR_PACK=1: the p-blocked k_pack_planes)
  static int pack_planes(const PackSrc& src, int R, int Kd, int RT, int ntiles, int nchunks, int kc, uint8_t* dst,
                         int KN, cudaStream_t s) {
    static const bool old_pack = getenv("GPIR_PACK") && atoi(getenv("GPIR_PACK")) == 1;
    if (old_pack) {
      dim3 g(KN / PK_P, (ntiles * RT + PK_R - 1) / PK_R, nchunks * (kc / PK_K));
      k_pack_planes<<<g, 256, 0, s>>>(src, R, Kd, RT, ntiles, nchunks, kc, dst);
      CKL();
      return 0;
    }
    static const int pw = getenv("GPIR_PACK") && atoi(getenv("GPIR_PACK")) == 16 ? 16 : 32;
    static bool attr = false;
    if (!attr) {
      CK(cudaFuncSetAttribute(k_pack_planes2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, Pk2<16>::SMEM));
      CK(cudaFuncSetAttribute(k_pack_planes2<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, Pk2<32>::SMEM));
      attr = true;
    }
    if (pw == 16) {
      dim3 g(KN / 16, (ntiles * RT + Pk2<16>::RR - 1) / Pk2<16>::RR, nchunks * (kc / PK_K));
      k_pack_planes2<16><<<g, 256, Pk2<16>::SMEM, s>>>(src, R, Kd, RT, ntiles, nchunks, kc, dst);
    } else {
      dim3 g(KN / 32, (ntiles * RT + Pk2<32>::RR - 1) / Pk2<32>::RR, nchunks * (kc / PK_K));
      k_pack_planes2<32><<<g, 256, Pk2<32>::SMEM, s>>>(src, R, Kd, RT, ntiles, nchunks, kc, dst);
    }
    CKL();
    return 0;
  }

  // RowSel execution plan for a (B, db) shape:
  //   kind 0: CUDA cores (k_rowsel_cc, d0 > 1024 or engine 1);
  //   kind 1: tensor cores, operands streamed per K chunk (k_rowsel_tc: M = 64 tiles, or d0 > 256);
  //   kind 2: tensor cores, A resident in TMEM (k_rowsel_tk: 2B > 64, d0 <= 256).
  // The A operand's byte-plane layout (a8) is fixed here so the last ExpandQuery
  // stage can write it directly (k_op_eq_mac_a8q, opt-in).
  struct RsPlan {
    int kind = 0;
    int M = 0, RA = 0, mtiles = 0, NT = 0, KC = 0, nchunks = 0, ntiles = 0, PST = 0;
    A8Desc a8{};
    size_t a8_bytes = 0;
  };
  static RsPlan rs_plan(gpir_ctx* c, int B, const gpir_db* db) {
    RsPlan r;
    const int KN = K * N;
    r.M = 2 * B;
    if (!tc_eligible(c, B, db)) return r;
    static const int tk_env = getenv("GPIR_TK") ? atoi(getenv("GPIR_TK")) : 1;
    const bool tk = db->compact || (tk_env && r.M > 64 && db->d0 <= 256);
    if (tk) {
      r.kind = 2;
      r.RA = 128;
      r.mtiles = (r.M + 127) / 128;
      r.NT = TK_NT;
      r.KC = ((int)db->d0 + 31) & ~31;
      r.nchunks = 1;
      r.ntiles = ((int)db->d1 + TK_NT - 1) / TK_NT;
    } else {
      r.kind = 1;
      r.RA = r.M <= 128 ? r.M : 128;
      r.mtiles = (r.M + r.RA - 1) / r.RA;
      const bool m64 = r.RA <= 64;
      static const int nt_env = getenv("GPIR_TC_NT") ? atoi(getenv("GPIR_TC_NT")) : 0;
      // N = 64 columns per tile when M = 64 (both TMEM accumulator buffers
      // still fit, lane-interleaved); M = 128 tiles use N = 32 with two
      // 7 x 32-column buffers so the epilogue overlaps the next item's MMAs
      r.NT = (nt_env == 32 || nt_env == 64) ? nt_env : (m64 && db->d1 >= 64 ? 64 : 32);
      static const int pst_env = getenv("GPIR_TC_PST") ? atoi(getenv("GPIR_TC_PST")) : 0;
      // p per staged epilogue flush: the staging buffer competes with the TMA
      // pipeline for shared memory, so the M64 x N64 tile stages 4 p (4 stages
      // in flight) rather than 8 (2 stages)
      r.PST = (!m64 && r.NT == 64)                               ? (pst_env == 2 ? 2 : 4)
              : (pst_env == 2 || pst_env == 4 || pst_env == 8) ? pst_env
              : m64                                            ? (r.NT == 64 ? 4 : 8)
                                                               : 4;
      r.KC = m64 ? 64 : 32;
      r.nchunks = ((int)db->d0 + r.KC - 1) / r.KC;
      r.ntiles = ((int)db->d1 + r.NT - 1) / r.NT;
    }
    // A8[p][c][mt][plane][g][row RA][16]
    const size_t blk = (size_t)4 * r.RA * r.KC;
    r.a8.base = nullptr;
    r.a8.s_mt = blk;
    r.a8.s_c = blk * r.mtiles;
    r.a8.s_p = r.a8.s_c * r.nchunks;
    r.a8.s_pl = (size_t)r.RA * r.KC;
    r.a8.s_g = (size_t)r.RA * 16;
    r.a8.G = r.KC / 16;
    r.a8.RA = r.RA;
    r.a8_bytes = r.a8.s_p * KN;
    return r;
  }

  // Column window of the capacity path (pipeline): the (B, d1) RowSel selection
  // and its P-major staging tensor are materialised per window of wd columns
  // when the whole selection exceeds the budget (GPIR_SEL_BUDGET_GIB, default
  // 16 GiB; GPIR_D1_WINDOW forces a width).  Windows are power-of-two column
  // ranges: the tournament pairs columns LSB-first inside each one
  // (src/planner.py:457-458), so the low log2(wd) ColTor stages run per window.
  static uint32_t window_d1(gpir_ctx* c, int B, const gpir_db* db, const RsPlan& rp) {
    const uint32_t d1 = db->d1;
    if (rp.kind != 2 || d1 <= TK_NT) return d1;
    static const long wenv = getenv("GPIR_D1_WINDOW") ? atol(getenv("GPIR_D1_WINDOW")) : 0;
    if (wenv >= TK_NT && (wenv & (wenv - 1)) == 0 && (uint32_t)wenv < d1) return (uint32_t)wenv;
    static const double genv = getenv("GPIR_SEL_BUDGET_GIB") ? atof(getenv("GPIR_SEL_BUDGET_GIB")) : 16.0;
    const size_t budget = c->sel_budget ? c->sel_budget : (size_t)(genv * (double)(1ull << 30));
    const size_t per_col = (size_t)B * CT * 4;
    uint32_t w = d1;
    while (w > (uint32_t)TK_NT && (size_t)w * per_col > budget) w >>= 1;
    return w;
  }

  // device workspace of one batch of B (bytes, excluding the DB and the key pool)
  static size_t ws_estimate(gpir_ctx* c, int B, const gpir_db* db) {
    const uint32_t total = leaves_of(db->d0, db->d1, ELL), bits = ilog2(db->d1);
    const RsPlan rp = rs_plan(c, B, db);
    const uint32_t wd = window_d1(c, B, db, rp), nw = db->d1 / wd;
    const size_t ctb = CT * 4;
    size_t per = 2 * (size_t)total * ctb + (size_t)3 * std::max<uint32_t>(bits, 1) * ELL * ctb +
                 (size_t)(wd + std::max<uint32_t>(wd / 2, nw) + wd / 4 + nw) * ctb;
    if (rp.kind == 2) per += (size_t)wd * ctb;  // P-major staging
    return (size_t)B * per + rp.a8_bytes + ((size_t)256 << 20);
  }

  // largest sub-batch that fits the free device memory (GPIR_MAX_BATCH overrides)
  static int max_subbatch(gpir_ctx* c, int B, const gpir_db* db) {
    static const int benv = getenv("GPIR_MAX_BATCH") ? atoi(getenv("GPIR_MAX_BATCH")) : 0;
    if (c->max_batch > 0) return std::min(B, c->max_batch);
    if (benv > 0) return std::min(B, benv);
    // cached per (db, B) while no device buffer changes (cudaMemGetInfo costs milliseconds per call)
    const uint64_t gen = g_alloc_gen.load();
    for (const auto& e : c->subbatch_cache)
      if (e.db == db && e.B == B && e.gen == gen) return e.bs;
    const int bs = max_subbatch_probe(c, B, db);
    if (c->subbatch_cache.size() > 32) c->subbatch_cache.clear();
    c->subbatch_cache.push_back({db, B, g_alloc_gen.load(), bs});
    return bs;
  }
  static int max_subbatch_probe(gpir_ctx* c, int B, const gpir_db* db) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return B;
    size_t held = 0;
    for (const DevBuf* b : {&c->ws_state0, &c->ws_state1, &c->ws_arows, &c->ws_sel, &c->ws_y, &c->ws_ct0, &c->ws_ct1,
                            &c->ws_crows, &c->ws_a8, &c->ws_part})
      held += b->bytes;
    const size_t margin = (size_t)4 << 30;
    const size_t budget = fr + held > margin ? fr + held - margin : 0;
    int bs = B;
    while (bs > 1 && ws_estimate(c, bs, db) > budget) bs = (bs + 1) / 2;
    return bs;
  }

  // DB byte planes D8[p][c][nt][plane][g][NT][16] in the plan's (NT, KC), packed once per layout
  static int ensure_d8(gpir_ctx* c, gpir_db* db, const RsPlan& r, cudaStream_t s) {
    const int KN = K * N;
    if (db->d8_nt == r.NT && db->d8_kc == r.KC) return 0;
    if (db->compact) FAIL(GPIR_INVALID_STATE, "compact database holds only the TMEM-resident RowSel layout");
    int rc;
    if ((rc = db->d8.ensure((size_t)KN * r.nchunks * r.ntiles * 4 * r.NT * r.KC))) return rc;
    CK(cudaMemsetAsync(db->d8.p, 0, db->d8.bytes, s));
    PackSrc ps{db->data.as<u32>(), (size_t)db->d0 * KN, 0, 1, (size_t)KN};
    if ((rc = pack_planes(ps, (int)db->d1, (int)db->d0, r.NT, r.ntiles, r.nchunks, r.KC, db->d8.as<uint8_t>(), KN, s)))
      return rc;
    db->d8_nt = r.NT;
    db->d8_kc = r.KC;
    // recorded graphs bake in the old byte-plane layout (the buffer may not have
    // been reallocated): retire them like any reallocation
    ++g_alloc_gen;
    return 0;
  }

  static int set_smem_attr(gpir_ctx* c, const void* kern, size_t smem) { return raise_smem_attr(c->device, kern, smem); }

  // RowSel: tensor-core path (byte-plane u8 GEMMs, rowsel_tc.cuh) when the
  // shape allows, else the CUDA-core kernel.  ev_mid (if non-null) is
  // recorded between operand packing and the GEMM.  a8_ready: the A operand
  // was already written in the plan's layout into ws_a8 (fused into the last
  // ExpandQuery stage).  want_il: the caller takes the ColTor pair-interleaved
  // output (kernels.cuh PAIRS_IL); *il_out reports whether it was produced.
  // win_d1 > 0 (k_rowsel_tk only): the column window [win_c0, win_c0 + win_d1) of
  // the DB (multiples of 32) into sel as a (B, win_d1) tensor -- the capacity path
  // runs RowSel and the low ColTor stages per window.
  static int rowsel(gpir_ctx* c, const u32* leaves, size_t a_b_words, int B, gpir_db* db, u32* sel,
                    cudaStream_t s, uint32_t* launches, cudaEvent_t ev_mid = nullptr, const RsPlan* plan = nullptr,
                    bool a8_ready = false, bool want_il = false, bool* il_out = nullptr, cudaEvent_t ev_y = nullptr,
                    int win_c0 = 0, int win_d1 = 0) {
    const int KN = K * N;
    int rc;
    if (il_out) *il_out = false;
    const RsPlan r = plan ? *plan : rs_plan(c, B, db);
    if (win_d1 && r.kind != 2) FAIL(GPIR_UNSUPPORTED, "column windows need the TMEM-resident RowSel");
    if (r.kind >= 1) {
      if ((rc = ensure_d8(c, db, r, s))) return rc;
      if ((rc = c->ws_a8.ensure(r.a8_bytes))) return rc;
      if (!a8_ready) {
        PackSrc pa{leaves, a_b_words, (size_t)KN, 2, 2 * (size_t)KN};
        if ((rc = pack_planes(pa, r.M, (int)db->d0, r.RA, r.mtiles, r.nchunks, r.KC, c->ws_a8.as<uint8_t>(), KN, s)))
          return rc;
        ++*launches;
      }
      if (ev_mid) CK(cudaEventRecord(ev_mid, s));
    }
    if (r.kind == 2) {
      // tensor-core GEMM into the P-major Y[p][m][n], then one transpose pass into the ciphertext layout
      const int wd1 = win_d1 ? win_d1 : (int)db->d1;
      const size_t ywords = (size_t)KN * r.M * wd1;
      if ((rc = c->ws_y.ensure(ywords * 4))) return rc;
      TkArgs ta;
      ta.A8 = c->ws_a8.as<uint8_t>();
      ta.D8 = db->d8.as<uint8_t>();
      ta.out = c->ws_y.as<u32>();
      ta.M = r.M;
      ta.mtiles = r.mtiles;
      ta.d1 = wd1;
      ta.ntiles = (wd1 + TK_NT - 1) / TK_NT;
      ta.nt0 = win_c0 / TK_NT;
      ta.ntiles_db = r.ntiles;
      ta.KN = KN;
      ta.logn = LOGN;
      ta.KC = r.KC;
      static const int pair_env = getenv("GPIR_TK_PAIR") ? atoi(getenv("GPIR_TK_PAIR")) : 0;
      ta.pair = (pair_env && r.mtiles % 2 == 0) ? 1 : 0;
      static const int aring_env = getenv("GPIR_TK_ARING") ? atoi(getenv("GPIR_TK_ARING")) : 0;
      ta.aring = (aring_env && !ta.pair) ? 1 : 0;
      ta.units = KN * (ta.pair ? r.mtiles / 2 : r.mtiles);
      const size_t slot = (size_t)128 * r.KC;
      const size_t fixed = (2 * TK_MAX_SLOTS + 16) * 8 + 16;
      ta.slots = std::min<int>(TK_MAX_SLOTS, (int)((226u * 1024u - fixed) / slot));
      const size_t smem = (size_t)ta.slots * slot + fixed;
      if ((rc = set_smem_attr(c, (const void*)k_rowsel_tk, smem))) return rc;
      const int grid = std::min(ta.units, c->num_sms);
      static const bool tprof_on = getenv("GPIR_TC_PROF") != nullptr;
      DevBuf tprof;
      ta.prof = nullptr;
      if (tprof_on) {
        if ((rc = tprof.ensure((size_t)grid * 8 * 8))) return rc;
        CK(cudaMemsetAsync(tprof.p, 0, tprof.bytes, s));
        ta.prof = tprof.as<unsigned long long>();
      }
      if (ta.pair) {  // clusters of 2 CTAs: the two row tiles of each p share the DB tiles by multicast
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * std::min(ta.units, c->num_sms / 2));
        cfg.blockDim = dim3(TK_THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, k_rowsel_tk, ta, c->tb));
      } else {
        k_rowsel_tk<<<grid, TK_THREADS, smem, s>>>(ta, c->tb);
      }
      CKL();
      if (tprof_on) {
        std::vector<unsigned long long> h((size_t)grid * 8);
        CK(cudaMemcpyAsync(h.data(), tprof.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double sum[8] = {0};
        for (int g = 0; g < grid; ++g)
          for (int k = 0; k < 8; ++k) sum[k] += (double)h[(size_t)g * 8 + k] / grid;
        fprintf(stderr, "[tk prof] avg cycles/CTA: mma_wait_drain+A %.0f mma_wait_data %.0f mma_issue_B %.0f epi_wait %.0f epi_work %.0f (data wait at unit starts %.0f, inside units %.0f)\n",
                sum[0], sum[1], sum[2], sum[3], sum[4], sum[5], sum[6]);
        tprof.release();
      }
      // the standard ciphertext layout: ColTor's first stage reads it faster than the pair-interleaved
      // one (config 3: ColTor 42.3 vs 45.2 ms, r2 A/B), at the same transpose cost
      static const int il_env = getenv("GPIR_PAIRS_IL") ? atoi(getenv("GPIR_PAIRS_IL")) : 0;
      const int il = (il_env && want_il && wd1 >= 2 && (wd1 & 1) == 0) ? 1 : 0;
      if (ev_y) CK(cudaEventRecord(ev_y, s));
      dim3 tg(KN / YT_P, r.M, (wd1 + YT_N - 1) / YT_N);
      k_y_to_cts<<<tg, 256, 0, s>>>(c->ws_y.as<u32>(), r.M, wd1, KN, sel, wd1, 0, il);
      CKL();
      *launches += 2;
      if (il_out) *il_out = il != 0;
      return 0;
    }
    if (r.kind == 1) {
      const bool m64 = r.RA <= 64;
      static const int ord_env = getenv("GPIR_TC_ORDER") ? atoi(getenv("GPIR_TC_ORDER")) : -1;
      const int NT = r.NT, PST = r.PST, KC = r.KC, RA = r.RA;
      TcArgs ta;
      ta.A8 = c->ws_a8.as<uint8_t>();
      ta.D8 = db->d8.as<uint8_t>();
      ta.out = sel;
      ta.M = r.M;
      ta.RA = RA;
      ta.mtiles = r.mtiles;
      ta.d1 = (int)db->d1;
      ta.ntiles = r.ntiles;
      ta.nchunks = r.nchunks;
      ta.KN = KN;
      ta.logn = LOGN;
      ta.items = KN * r.ntiles * r.mtiles;
      ta.nt_outer = ord_env >= 0 ? ord_env : 0;
      const uint32_t stage_bytes = ((4u * RA * KC + 4u * NT * KC) + 127u) & ~127u;
      const size_t outbuf = (size_t)PST * RA * (NT + 1) * 4;
      const size_t fixed = 4096 + outbuf + 2 * TC_MAX_STAGES * 8 + 4 * 8 + 16;
      ta.stages = std::max(2, std::min<int>(TC_MAX_STAGES, (int)((226u * 1024u - fixed) / stage_bytes)));
      const size_t smem = (size_t)ta.stages * stage_bytes + fixed;
      const int grid = std::min(KN / PST, c->num_sms);
      static const bool prof_on = getenv("GPIR_TC_PROF") != nullptr;
      DevBuf profbuf;
      ta.prof = nullptr;
      if (prof_on) {
        if ((rc = profbuf.ensure((size_t)grid * 8 * 8))) return rc;
        CK(cudaMemsetAsync(profbuf.p, 0, profbuf.bytes, s));
        ta.prof = profbuf.as<unsigned long long>();
      }
      auto kern = m64 ? (NT == 64 ? (PST == 8   ? k_rowsel_tc<64, true, 8, 64>
                                     : PST == 4 ? k_rowsel_tc<64, true, 4, 64>
                                                : k_rowsel_tc<64, true, 2, 64>)
                                  : (PST == 8   ? k_rowsel_tc<32, true, 8, 64>
                                     : PST == 4 ? k_rowsel_tc<32, true, 4, 64>
                                                : k_rowsel_tc<32, true, 2, 64>))
                      : (NT == 64 ? (PST == 2 ? k_rowsel_tc<64, false, 2, 32> : k_rowsel_tc<64, false, 4, 32>)
                                  : (PST == 2   ? k_rowsel_tc<32, false, 2, 32>
                                     : PST == 4 ? k_rowsel_tc<32, false, 4, 32>
                                                : k_rowsel_tc<32, false, 8, 32>));
      if ((rc = set_smem_attr(c, (const void*)kern, smem))) return rc;
      kern<<<grid, TC_THREADS, smem, s>>>(ta, c->tb);
      CKL();
      if (ev_y) CK(cudaEventRecord(ev_y, s));
      if (prof_on) {
        std::vector<unsigned long long> h((size_t)grid * 8);
        CK(cudaMemcpyAsync(h.data(), profbuf.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double sum[8] = {0};
        for (int g = 0; g < grid; ++g)
          for (int k = 0; k < 8; ++k) sum[k] += (double)h[(size_t)g * 8 + k] / grid;
        fprintf(stderr, "[tc prof] avg cycles/CTA: mma_wait_tmem %.0f mma_wait_data %.0f mma_issue %.0f epi_wait %.0f epi_work %.0f (data wait at unit starts %.0f, inside units %.0f)\n",
                sum[0], sum[1], sum[2], sum[3], sum[4], sum[5], sum[6]);
        profbuf.release();
      }
      ++*launches;
      return 0;
    }
    const int mt = (2 * B + RS_MT - 1) / RS_MT, nt = ((int)db->d1 + RS_NT - 1) / RS_NT;
    dim3 grid(mt * nt, KN / 32);
    static bool attr = false;
    if (!attr) {
      CK(cudaFuncSetAttribute(k_rowsel_cc, cudaFuncAttributeMaxDynamicSharedMemorySize, RS_SMEM));
      attr = true;
    }
    if (ev_mid) CK(cudaEventRecord(ev_mid, s));
    k_rowsel_cc<<<grid, 256, RS_SMEM, s>>>(leaves, a_b_words, 2 * B, db->data.as<u32>(), (int)db->d0, (int)db->d1,
                                           sel, KN, LOGN, c->tb);
    CKL();
    if (ev_y) CK(cudaEventRecord(ev_y, s));
    ++*launches;
    return 0;
  }

  static RowsDesc evk_rows(gpir_ctx* c, int t, const int* kslot) {
    RowsDesc r;
    r.lo = c->evk_pool.as<u32>() + (size_t)t * ELL * CT;
    r.lo_b = (size_t)c->key_stages * ELL * CT;
    r.hi = r.lo;
    r.hi_b = r.lo_b;
    r.slot = kslot;
    return r;
  }
  static RowsDesc skrgsw_rows(gpir_ctx* c, const int* kslot) {
    RowsDesc r;
    r.lo = c->rgsw_pool.as<u32>();
    r.lo_b = 2 * (size_t)ELL * CT;
    r.hi = r.lo + (size_t)ELL * CT;
    r.hi_b = r.lo_b;
    r.slot = kslot;
    return r;
  }

  // ColTor RGSW rows of bits [0, nb): a-digit rows from `arows` (query
  // stride arows_b words, ELL rows per bit) and b-digit rows = the column
  // leaves `cols` (query stride cols_b), folded (k_fold_rows) into ws_crows
  // as (B, nb, 2 ELL) row groups.
  static int fold_coltor(gpir_ctx* c, int B, uint32_t nb, const u32* arows, size_t arows_b, const u32* cols,
                         size_t cols_b, cudaStream_t s) {
    if (!nb) return 0;
    u32* dst = c->ws_crows.as<u32>();
    const size_t db = (size_t)nb * 2 * ELL * CT, dg = 2 * (size_t)ELL * CT;
    int rc;
    if ((rc = fold_rows(c, arows, dst, B, (int)nb, arows_b, (size_t)ELL * CT, db, dg, s))) return rc;
    return fold_rows(c, cols, dst + (size_t)ELL * CT, B, (int)nb, cols_b, (size_t)ELL * CT, db, dg, s);
  }
  static RowsDesc coltor_rows(gpir_ctx* c, uint32_t nb, uint32_t j) {
    RowsDesc r;
    r.lo = c->ws_crows.as<u32>() + (size_t)j * 2 * ELL * CT;
    r.lo_b = (size_t)nb * 2 * ELL * CT;
    r.hi = r.lo + (size_t)ELL * CT;
    r.hi_b = r.lo_b;
    r.slot = nullptr;
    return r;
  }

  // expansion of B brv queries (in ws_state0 as (B,1)) -> leaves pointer (B, total)
  // a8f: the RowSel A-operand layout to fuse into the last stage (or null);
  // *fused reports whether the last stage wrote it (operation-level last stage,
  // d0 % 16 == 0, d0 <= its node count per query)
  static int expand_all(gpir_ctx* c, int B, uint32_t total, const uint8_t* eq_modes, uint32_t n_eq,
                        const int* kslot, u32** leaves_out, cudaStream_t s, uint32_t* launches,
                        const A8Desc* a8f = nullptr, int d0 = 0, bool* fused = nullptr) {
    const uint32_t stages = stages_of(total);
    u32* cur = c->ws_state0.as<u32>();
    u32* nxt = c->ws_state1.as<u32>();
    if (fused) *fused = false;
    for (uint32_t t = 0; t < stages; ++t) {
      const int C = (int)std::min<uint32_t>(1u << t, total);
      const int Cout = (int)std::min<uint32_t>(2u << t, total);
      const int mode = (eq_modes && t < n_eq) ? eq_modes[t] : default_mode(B * C);
      const bool fuse = a8f && t + 1 == stages && mode == 0 && d0 > 0 && d0 % 16 == 0 && d0 <= C && C % 16 == 0;
      int rc = expand_stage(c, cur, B, C, nxt, Cout, (int)t, evk_rows(c, (int)t, kslot), mode, s, launches,
                            fuse ? a8f : nullptr, d0);
      if (fuse && fused) *fused = true;
      if (rc) return rc;
      g_sprof.mark(s, "eq" + std::to_string(t) + " " + "oFSH"[mode & 3], 0, (int)t, mode, (uint32_t)(B * C));
      std::swap(cur, nxt);
    }
    *leaves_out = cur;
    return 0;
  }

  // B200 hybrid rule (measured per stage, profiles/r1_plans.md, r1g_plans.md):
  // ExpandQuery runs operation-level at every stage since the MAC kernel
  // batches 8 nodes per thread over their shared key rows (k_op_eq_mac_nb);
  // ColTor and RGSW assembly switch to the stage-level executor (mode 3:
  // operation-level iNTT + Dcp feeding the fused digit-NTT + key-switch MAC
  // kernel) from 64 ciphertexts.  The single-kernel node-fused executor
  // (mode 1) is limited to 2 CTAs/SM by its 112 KiB of shared memory and is
  // never the faster choice on B200.
  static int eq_default(size_t nodes) { return nodes >= kEqStageNodes ? 3 : 0; }
  static int xp_default(size_t cts) { return cts >= kXpStageCts ? 3 : 0; }
  static int default_mode(size_t nodes) { return eq_default(nodes); }

  // wd: the RowSel column window (d1 unless the capacity path splits the columns)
  static int ensure_ws(gpir_ctx* c, int B, uint32_t total, uint32_t d1, uint32_t bits, uint32_t wd = 0) {
    int rc;
    const size_t ctb = CT * 4;
    if (!wd) wd = d1;
    const uint32_t nw = d1 / wd;
    if ((rc = c->ws_state0.ensure((size_t)B * total * ctb))) return rc;
    if ((rc = c->ws_state1.ensure((size_t)B * total * ctb))) return rc;
    if ((rc = c->ws_arows.ensure((size_t)B * std::max<uint32_t>(bits, 1) * ELL * ctb))) return rc;
    if ((rc = c->ws_sel.ensure((size_t)B * wd * ctb))) return rc;
    if ((rc = c->ws_ct0.ensure((size_t)B * std::max<uint32_t>(std::max(wd / 2, nw / 2), 1) * ctb))) return rc;
    if ((rc = c->ws_ct1.ensure((size_t)B * std::max<uint32_t>(std::max(wd / 4, nw / 4), 1) * ctb))) return rc;
    if ((rc = c->ws_kslot.ensure((size_t)B * 4))) return rc;
    if ((rc = c->ws_crows.ensure((size_t)B * std::max<uint32_t>(bits, 1) * 2 * ELL * ctb))) return rc;
    return 0;
  }

  // stats: an event recorded now (nullptr when stats are off)
  static cudaEvent_t mark(gpir_ctx* c, cudaStream_t s, bool on) {
    if (!on) return nullptr;
    cudaEvent_t e = c->ev_next();
    cudaEventRecord(e, s);
    return e;
  }
  static void span(gpir_ctx* c, int phase, cudaEvent_t a, cudaEvent_t b) {
    if (a && b) c->plog.push_back({phase, a, b});
  }

  // Full pipeline on device, brv queries already in ws_state0 as (B, 1).
  // Runs expansion over (d0, d1_tree), RGSW assembly for all log2(d1_tree)
  // bits, RowSel on db, and the low log2(db->d1) ColTor stages; returns the
  // pointer to the (B, 1) brv result and the leaves / a-rows for the caller.
  // keep_rows: the caller reads the u32 row leaves afterwards (no fused A-operand write)
  static int pipeline(gpir_ctx* c, gpir_db* db, uint32_t d1_tree, int B, const uint8_t* eq_modes, uint32_t n_eq,
                      const uint8_t* ct_modes, uint32_t n_ct, const int* kslot, cudaStream_t s, gpir_stats* st,
                      u32** result, u32** leaves_out, bool keep_rows = false) {
    const uint32_t d0 = db->d0, d1 = db->d1;
    const uint32_t total = leaves_of(d0, d1_tree, ELL);
    const uint32_t bits_tree = ilog2(d1_tree), bits = ilog2(d1);
    uint32_t launches = 0;
    int rc;
    const bool on = st != nullptr;
    cudaEvent_t t_start = mark(c, s, on);
    g_sprof.begin(c->stage_timing != 0);
    g_sprof.mark(s, "start");
    u32* leaves = nullptr;
    // RowSel plan first: its A-operand layout is written by the last ExpandQuery stage
    RsPlan rp = rs_plan(c, B, db);
    A8Desc a8f = rp.a8;
    bool fused = false;
    // The A operand written by the last ExpandQuery stage (k_op_eq_mac_a8q) is opt-in
    // (GPIR_FUSE_A8=1): its one-slot-per-thread MAC (coalesced byte-plane writes need
    // lanes over queries) costs more than the separate coalesced pack it replaces
    // (config 2: ExpandQuery +1.05 vs pack 0.46 ms, config 3: +4.6 vs 1.84 ms, r2 A/B)
    static const bool fuse_env = getenv("GPIR_FUSE_A8") && atoi(getenv("GPIR_FUSE_A8")) != 0;
    const bool fuse_ok = rp.kind >= 1 && fuse_env && !keep_rows;
    if (fuse_ok) {
      if ((rc = c->ws_a8.ensure(rp.a8_bytes))) return rc;
      a8f.base = c->ws_a8.as<uint8_t>();
    }
    if ((rc = expand_all(c, B, total, eq_modes, n_eq, kslot, &leaves, s, &launches, fuse_ok ? &a8f : nullptr,
                         (int)d0, &fused)))
      return rc;
    cudaEvent_t t_eq = mark(c, s, on);
    span(c, 0, t_start, t_eq);
    // RGSW assembly (src/protocol.py:383-409): a-rows = col_cts ⊡ RGSW(s)
    if (bits_tree > 0) {
      const int M = (int)(bits_tree * ELL);
      static const int rgsw_env = getenv("GPIR_RGSW_MODE") ? atoi(getenv("GPIR_RGSW_MODE")) : -1;
      const int mode = rgsw_env >= 0 ? rgsw_env : xp_default((size_t)B * M);
      if ((rc = ext_product(c, leaves + (size_t)d0 * CT, total, B, M, 0, c->ws_arows.as<u32>(), (size_t)M,
                            skrgsw_rows(c, kslot), mode, s, &launches)))
        return rc;
    }
    cudaEvent_t t_rgsw = mark(c, s, on);
    span(c, 1, t_eq, t_rgsw);
    g_sprof.mark(s, "rgsw", 1, 0, xp_default((size_t)B * bits_tree * ELL), (uint32_t)(B * bits_tree * ELL));
    const uint32_t wd = window_d1(c, B, db, rp);
    if (wd < d1) {  // capacity path: RowSel + the low log2(wd) ColTor stages per column window
      if ((rc = fold_coltor(c, B, bits, c->ws_arows.as<u32>(), (size_t)bits_tree * ELL * CT,
                            leaves + (size_t)d0 * CT, (size_t)total * CT, s)))
        return rc;
      const uint32_t nw = d1 / wd, wbits = ilog2(wd);
      if ((rc = c->ws_part.ensure((size_t)B * nw * CT * 4))) return rc;
      u32* bufs[2] = {c->ws_ct0.as<u32>(), c->ws_ct1.as<u32>()};
      cudaEvent_t t_w = t_rgsw;
      for (uint32_t w = 0; w < nw; ++w) {
        bool il = false;
        cudaEvent_t e_mid = on ? c->ev_next() : nullptr, e_y = on ? c->ev_next() : nullptr;
        if ((rc = rowsel(c, leaves, (size_t)total * CT, B, db, c->ws_sel.as<u32>(), s, &launches, e_mid, &rp,
                         fused || w > 0, true, &il, e_y, (int)(w * wd), (int)wd)))
          return rc;
        cudaEvent_t t_tr = mark(c, s, on);
        span(c, 2, t_w, e_mid);
        span(c, 3, e_mid, e_y);
        span(c, 4, e_y, t_tr);
        u32* cur = c->ws_sel.as<u32>();
        for (uint32_t j = 0; j < wbits; ++j) {
          const int C = (int)(wd >> j);
          const RowsDesc r = coltor_rows(c, bits, j);
          const int mode = (ct_modes && j < n_ct) ? ct_modes[j] : xp_default((size_t)B * C / 2);
          const bool last = j + 1 == wbits;
          u32* dst = last ? c->ws_part.as<u32>() + (size_t)w * CT : bufs[j & 1];
          if ((rc = ext_product(c, cur, (size_t)C, B, C / 2, (j == 0 && il) ? PAIRS_IL : 1, dst,
                                last ? (size_t)nw : (size_t)C / 2, r, mode, s, &launches)))
            return rc;
          cur = dst;
        }
        t_w = mark(c, s, on);
        span(c, 5, t_tr, t_w);
      }
      g_sprof.mark(s, "rowsel+coltor low (windows of " + std::to_string(wd) + ")", 2, 0, 0, (uint32_t)B);
      u32* cur = c->ws_part.as<u32>();
      for (uint32_t j = wbits; j < bits; ++j) {
        const int C = (int)(d1 >> j);
        const RowsDesc r = coltor_rows(c, bits, j);
        const int mode = (ct_modes && j < n_ct) ? ct_modes[j] : xp_default((size_t)B * C / 2);
        u32* dst = bufs[j & 1];
        if ((rc = ext_product(c, cur, (size_t)C, B, C / 2, 1, dst, (size_t)C / 2, r, mode, s, &launches))) return rc;
        g_sprof.mark(s, "coltor" + std::to_string(j) + " " + "oFSH"[mode & 3], 3, (int)j, mode, (uint32_t)(B * C / 2));
        cur = dst;
      }
      span(c, 5, t_w, mark(c, s, on));
      g_sprof.flush(&c->last_stages);
      *result = cur;
      if (leaves_out) *leaves_out = leaves;
      if (st) st->launches += launches;
      return 0;
    }
    bool il = false;
    cudaEvent_t e_mid = on ? c->ev_next() : nullptr, e_y = on ? c->ev_next() : nullptr;
    if ((rc = rowsel(c, leaves, (size_t)total * CT, B, db, c->ws_sel.as<u32>(), s, &launches, e_mid, &rp, fused,
                     bits > 0, &il, e_y)))
      return rc;
    cudaEvent_t t_rs = mark(c, s, on);
    span(c, 2, t_rgsw, e_mid);
    span(c, 3, e_mid, e_y);
    span(c, 4, e_y, t_rs);
    g_sprof.mark(s, "rowsel+pack", 2, 0, 0, (uint32_t)B);
    // ColTor (src/protocol.py:542-573): LSB-first pairs
    if ((rc = fold_coltor(c, B, bits, c->ws_arows.as<u32>(), (size_t)bits_tree * ELL * CT, leaves + (size_t)d0 * CT,
                          (size_t)total * CT, s)))
      return rc;
    u32* cur = c->ws_sel.as<u32>();
    u32* bufs[2] = {c->ws_ct0.as<u32>(), c->ws_ct1.as<u32>()};
    for (uint32_t j = 0; j < bits; ++j) {
      const int C = (int)(d1 >> j);
      const RowsDesc r = coltor_rows(c, bits, j);
      const int mode = (ct_modes && j < n_ct) ? ct_modes[j] : xp_default((size_t)B * C / 2);
      u32* dst = bufs[j & 1];
      if ((rc = ext_product(c, cur, (size_t)C, B, C / 2, (j == 0 && il) ? PAIRS_IL : 1, dst, (size_t)C / 2, r, mode, s,
                            &launches)))
        return rc;
      g_sprof.mark(s, "coltor" + std::to_string(j) + " " + "oFSH"[mode & 3], 3, (int)j, mode, (uint32_t)(B * C / 2));
      cur = dst;
    }
    span(c, 5, t_rs, mark(c, s, on));
    g_sprof.flush(&c->last_stages);
    *result = cur;
    if (leaves_out) *leaves_out = leaves;
    if (st) st->launches += launches;
    return 0;
  }

  static int answer_dev(gpir_ctx* c, gpir_db* db, const u32* d_q, const int32_t* slots, int B,
                        const uint8_t* eq_modes, uint32_t n_eq, const uint8_t* ct_modes, uint32_t n_ct, u32* d_out,
                        cudaStream_t s, gpir_stats* st) {
    const uint32_t d0 = db->d0, d1 = db->d1;
    const uint32_t total = leaves_of(d0, d1, ELL), bits = ilog2(d1);
    int rc;
    if ((rc = check_keys(c, slots, B, stages_of(total), bits > 0))) return rc;
    // batches larger than the free memory allows run as consecutive sub-batches
    // (each reads the DB once more in RowSel; responses do not depend on batch composition)
    const int Bs = max_subbatch(c, B, db);
    if ((rc = ensure_ws(c, Bs, total, d1, bits, window_d1(c, Bs, db, rs_plan(c, Bs, db))))) return rc;
    if ((rc = c->ws_kslot.ensure((size_t)B * 4))) return rc;
    c->evp_used = 0;
    c->plog.clear();
    if (st) CK(cudaEventRecord(c->ev[0], s));
    CK(cudaMemcpyAsync(c->ws_kslot.p, slots, (size_t)B * 4, cudaMemcpyHostToDevice, s));
    auto body = [&]() -> int {
      int r;
      for (int b0 = 0; b0 < B; b0 += Bs) {
        const int nb = std::min(Bs, B - b0);
        const size_t off = (size_t)b0 * CT;
        if ((r = bitrev_rows(c, d_q + off, c->ws_state0.as<u32>(), (size_t)nb * 2 * K, s))) return r;
        u32* res = nullptr;
        if (st) st->launches += 2;
        if ((r = pipeline(c, db, d1, nb, eq_modes, n_eq, ct_modes, n_ct, c->ws_kslot.as<int>() + b0, s, st, &res,
                          nullptr)))
          return r;
        if ((r = bitrev_rows(c, res, d_out + off, (size_t)nb * 2 * K, s))) return r;
      }
      return 0;
    };
    // graph replay: not with per-phase stats or stage timing (their events and syncs), and
    // not while the caller is itself capturing the stream (the launches then go into its graph)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(s, &cap));
    if (c->use_graph && !st && !c->stage_timing && !g_sprof.env && cap == cudaStreamCaptureStatusNone) {
      std::vector<uint8_t> modes(34, 0);
      modes[0] = (uint8_t)n_eq;
      modes[1] = (uint8_t)n_ct;
      for (uint32_t j = 0; j < n_eq && j < 16 && eq_modes; ++j) modes[2 + j] = eq_modes[j];
      for (uint32_t j = 0; j < n_ct && j < 16 && ct_modes; ++j) modes[18 + j] = ct_modes[j];
      const uint64_t gen = g_alloc_gen.load();
      gpir_ctx::GraphEntry* e = nullptr;
      for (auto& g : c->graphs)
        if (g.db == db && g.dq == d_q && g.dout == d_out && g.B == B && g.gen == gen && g.modes == modes) e = &g;
      if (!e) {
        if (c->graphs.size() >= 16) {
          if (c->graphs.front().exec) cudaGraphExecDestroy(c->graphs.front().exec);
          c->graphs.erase(c->graphs.begin());
        }
        gpir_ctx::GraphEntry ne;
        ne.db = db, ne.dq = d_q, ne.dout = d_out, ne.B = B, ne.gen = gen, ne.modes = modes, ne.state = 1;
        c->graphs.push_back(ne);
        return body();  // first call eager
      }
      if (e->state == 2) {
        CK(cudaGraphLaunch(e->exec, s));
        return 0;
      }
      if (e->state == 1) {  // capture, instantiate, launch; on any failure stay eager for this key
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        const int r = body();
        const cudaError_t ce = cudaStreamEndCapture(s, &g);
        if (!r && ce == cudaSuccess && g && cudaGraphInstantiate(&e->exec, g, 0) == cudaSuccess) {
          cudaGraphDestroy(g);
          e->state = 2;
          CK(cudaGraphLaunch(e->exec, s));
          return 0;
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        e->state = -1;
        e->exec = nullptr;
      }
    }
    if ((rc = body())) return rc;
    if (st) {
      CK(cudaEventRecord(c->ev[6], s));
      CK(cudaEventSynchronize(c->ev[6]));
      float a;
      sum_phases(c, st);
      cudaEventElapsedTime(&a, c->ev[0], c->ev[6]);
      st->ms_total = a;
    }
    return 0;
  }

  // phase sums of the logged intervals (all windows and sub-batches of the call)
  static void sum_phases(gpir_ctx* c, gpir_stats* st) {
    double ph[6] = {0, 0, 0, 0, 0, 0};
    for (const auto& iv : c->plog) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, iv.a, iv.b) == cudaSuccess) ph[iv.phase] += ms;
    }
    st->ms_expand = (float)ph[0];
    st->ms_rgsw = (float)ph[1];
    st->ms_rowsel = (float)(ph[2] + ph[3] + ph[4]);
    st->ms_rowsel_kernel = (float)ph[3];
    st->ms_rowsel_transpose = (float)ph[4];
    st->ms_coltor = (float)ph[5];
    c->plog.clear();
    c->evp_used = 0;
    cudaGetLastError();  // an interval that could not be timed must not surface as a later launch error
  }

  static int check_keys(gpir_ctx* c, const int32_t* slots, int B, uint32_t stages, bool need_rgsw) {
    for (int b = 0; b < B; ++b) {
      const int sl = slots[b];
      if (sl < 0 || (uint32_t)sl >= c->key_slots || c->slot_stages[sl] < 0)
        FAIL(GPIR_INVALID_STATE, "no uploaded keys for key slot " + std::to_string(sl));
      if ((uint32_t)c->slot_stages[sl] < stages)
        FAIL(GPIR_INVALID_STATE, "key slot " + std::to_string(sl) + " has too few evaluation keys");
      if (need_rgsw && !c->slot_rgsw[sl])
        FAIL(GPIR_INVALID_STATE, "key slot " + std::to_string(sl) + " has no RGSW of the secret");
    }
    return 0;
  }

  // sharded: expansion over (d0, d1_total), local rowsel + low ColTor on db's columns
  static int shard_answer(gpir_ctx* c, gpir_db* db, uint32_t d1_total, const u32* d_q, const int32_t* slots,
                          int B, u32* d_partials, u32* d_high, cudaStream_t s, gpir_stats* st) {
    const uint32_t d0 = db->d0;
    const uint32_t total = leaves_of(d0, d1_total, ELL);
    const uint32_t bits_tree = ilog2(d1_total), bits = ilog2(db->d1);
    if (d1_total < db->d1 || (d1_total & (d1_total - 1))) FAIL(GPIR_INVALID_ARGUMENT, "bad d1_total");
    int rc;
    if ((rc = check_keys(c, slots, B, stages_of(total), bits_tree > 0))) return rc;
    if ((rc = ensure_ws(c, B, total, db->d1, bits_tree))) return rc;
    CK(cudaMemcpyAsync(c->ws_kslot.p, slots, (size_t)B * 4, cudaMemcpyHostToDevice, s));
    if ((rc = bitrev_rows(c, d_q, c->ws_state0.as<u32>(), (size_t)B * 2 * K, s))) return rc;
    u32* res = nullptr;
    u32* leaves = nullptr;
    c->evp_used = 0;
    c->plog.clear();
    if ((rc = pipeline(c, db, d1_total, B, nullptr, 0, nullptr, 0, c->ws_kslot.as<int>(), s, st, &res, &leaves)))
      return rc;
    if (st) {
      CK(cudaStreamSynchronize(s));
      sum_phases(c, st);
    }
    if ((rc = bitrev_rows(c, res, d_partials, (size_t)B * 2 * K, s))) return rc;
    if (d_high) {
      const uint32_t nh = bits_tree - bits;
      for (int b = 0; b < B; ++b)
        for (uint32_t h = 0; h < nh; ++h) {
          const uint32_t j = bits + h;
          u32* dst = d_high + (((size_t)b * nh + h) * 2 * ELL) * CT;
          const u32* a_rows = c->ws_arows.as<u32>() + ((size_t)b * bits_tree + j) * ELL * CT;
          const u32* b_rows = leaves + ((size_t)b * total + d0 + j * ELL) * CT;
          if ((rc = bitrev_rows(c, a_rows, dst, (size_t)ELL * 2 * K, s))) return rc;
          if ((rc = bitrev_rows(c, b_rows, dst + (size_t)ELL * CT, (size_t)ELL * 2 * K, s))) return rc;
        }
    }
    return 0;
  }

  // ---- row-sharded pipeline (D0 shards, modular-add combine) -----------------------
  // expand the rank's own queries over the full (d0, d1) tree, assemble their
  // RGSWs, and export the row leaves (B, d0, ct) in the internal brv layout.
  static int sh_expand(gpir_ctx* c, uint32_t d0, uint32_t d1, const u32* d_q, const int32_t* slots, int B,
                       u32* d_rows, cudaStream_t s) {
    const uint32_t total = leaves_of(d0, d1, ELL), bits = ilog2(d1);
    int rc;
    if ((rc = check_keys(c, slots, B, stages_of(total), bits > 0))) return rc;
    // expansion workspace only: the selection / tournament buffers are sized by the steps that use them
    const size_t ctb = CT * 4;
    if ((rc = c->ws_state0.ensure((size_t)B * total * ctb))) return rc;
    if ((rc = c->ws_state1.ensure((size_t)B * total * ctb))) return rc;
    if ((rc = c->ws_arows.ensure((size_t)B * std::max<uint32_t>(bits, 1) * ELL * ctb))) return rc;
    if ((rc = c->ws_crows.ensure((size_t)B * std::max<uint32_t>(bits, 1) * 2 * ELL * ctb))) return rc;
    if ((rc = c->ws_kslot.ensure((size_t)B * 4))) return rc;
    CK(cudaMemcpyAsync(c->ws_kslot.p, slots, (size_t)B * 4, cudaMemcpyHostToDevice, s));
    if ((rc = bitrev_rows(c, d_q, c->ws_state0.as<u32>(), (size_t)B * 2 * K, s))) return rc;
    uint32_t launches = 0;
    u32* leaves = nullptr;
    if ((rc = expand_all(c, B, total, nullptr, 0, c->ws_kslot.as<int>(), &leaves, s, &launches))) return rc;
    if (bits > 0) {
      const int M = (int)(bits * ELL);
      if ((rc = ext_product(c, leaves + (size_t)d0 * CT, total, B, M, 0, c->ws_arows.as<u32>(), (size_t)M,
                            skrgsw_rows(c, c->ws_kslot.as<int>()), xp_default((size_t)B * M), s, &launches)))
        return rc;
    }
    CK(cudaMemcpy2DAsync(d_rows, (size_t)d0 * CT * 4, leaves, (size_t)total * CT * 4, (size_t)d0 * CT * 4, B,
                         cudaMemcpyDeviceToDevice, s));
    c->sh_leaves = leaves;
    c->sh_B = B;
    c->sh_d0 = d0;
    c->sh_d1 = d1;
    c->sh_total = total;
    return 0;
  }

  // ColTor for the session's own queries from combined RowSel sums (int32,
  // brv, sum of shard partials < n q): reduce mod q, run all log2(d1) stages.
  // RGSW rows of column bits [lo, hi) for the session's own queries (after
  // sh_expand), natural order, as (B, hi - lo, 2 ELL) ciphertexts: a-digit rows
  // from the RGSW assembly, b-digit rows = the column leaves (src/protocol.py:383-409).
  static int sh_rgsw(gpir_ctx* c, uint32_t lo, uint32_t hi, u32* d_out, cudaStream_t s) {
    if (!c->sh_leaves) FAIL(GPIR_INVALID_STATE, "gpir_sharded_expand must precede gpir_sharded_rgsw");
    const uint32_t bits = ilog2(c->sh_d1), B = c->sh_B, total = c->sh_total, d0 = c->sh_d0;
    if (lo > hi || hi > bits) FAIL(GPIR_INVALID_ARGUMENT, "bit range outside the session's tournament");
    const uint32_t nb = hi - lo;
    int rc;
    for (uint32_t b = 0; b < B; ++b)
      for (uint32_t h = 0; h < nb; ++h) {
        const uint32_t j = lo + h;
        u32* dst = d_out + (((size_t)b * nb + h) * 2 * ELL) * CT;
        const u32* a_rows = c->ws_arows.as<u32>() + ((size_t)b * bits + j) * ELL * CT;
        const u32* b_rows = c->sh_leaves + ((size_t)b * total + d0 + j * ELL) * CT;
        if ((rc = bitrev_rows(c, a_rows, dst, (size_t)ELL * 2 * K, s))) return rc;
        if ((rc = bitrev_rows(c, b_rows, dst + (size_t)ELL * CT, (size_t)ELL * 2 * K, s))) return rc;
      }
    return 0;
  }

  static int sh_coltor(gpir_ctx* c, u32* d_sums, int B, u32* d_out, cudaStream_t s) {
    if (!c->sh_leaves || (uint32_t)B != c->sh_B) FAIL(GPIR_INVALID_STATE, "gpir_sharded_expand must precede gpir_sharded_coltor");
    const uint32_t d1 = c->sh_d1, bits = ilog2(d1), total = c->sh_total, d0 = c->sh_d0;
    const size_t rows = (size_t)B * d1 * 2 * K;
    int rc0;
    if ((rc0 = c->ws_ct0.ensure(std::max(c->ws_ct0.bytes, (size_t)B * std::max<uint32_t>(d1 / 2, 1) * CT * 4))))
      return rc0;
    if ((rc0 = c->ws_ct1.ensure(std::max(c->ws_ct1.bytes, (size_t)B * std::max<uint32_t>(d1 / 4, 1) * CT * 4))))
      return rc0;
    k_mod_rows<<<(unsigned)((rows * N + 255) / 256), 256, 0, s>>>(d_sums, rows, LOGN, K, c->tb);
    CKL();
    u32* cur = d_sums;
    u32* bufs[2] = {c->ws_ct0.as<u32>(), c->ws_ct1.as<u32>()};
    uint32_t launches = 0;
    int rc;
    if ((rc = fold_coltor(c, B, bits, c->ws_arows.as<u32>(), (size_t)bits * ELL * CT, c->sh_leaves + (size_t)d0 * CT,
                          (size_t)total * CT, s)))
      return rc;
    for (uint32_t j = 0; j < bits; ++j) {
      const int C = (int)(d1 >> j);
      const RowsDesc r = coltor_rows(c, bits, j);
      u32* dst = bufs[j & 1];
      if ((rc = ext_product(c, cur, (size_t)C, B, C / 2, 1, dst, (size_t)C / 2, r, xp_default((size_t)B * C / 2), s,
                            &launches)))
        return rc;
      cur = dst;
    }
    return bitrev_rows(c, cur, d_out, (size_t)B * 2 * K, s);
  }

  static int coltor_dev(gpir_ctx* c, const u32* d_cts, int B, int C, const u32* d_rgsw, u32* d_out, cudaStream_t s) {
    const uint32_t bits = ilog2((uint32_t)C);
    int rc;
    uint32_t launches = 0;
    // brv copies: cts -> ws_state0, rgsw -> ws_state1 (layout (B, bits, 2 ELL))
    if ((rc = c->ws_state0.ensure(std::max<size_t>(c->ws_state0.bytes, (size_t)B * C * CT * 4)))) return rc;
    if ((rc = c->ws_io0.ensure((size_t)B * std::max<uint32_t>(bits, 1) * 2 * ELL * CT * 4))) return rc;
    if ((rc = c->ws_ct0.ensure(std::max<size_t>(c->ws_ct0.bytes, (size_t)B * std::max(C / 2, 1) * CT * 4)))) return rc;
    if ((rc = c->ws_ct1.ensure(std::max<size_t>(c->ws_ct1.bytes, (size_t)B * std::max(C / 4, 1) * CT * 4)))) return rc;
    if ((rc = bitrev_rows(c, d_cts, c->ws_state0.as<u32>(), (size_t)B * C * 2 * K, s))) return rc;
    if (bits) {
      if ((rc = bitrev_rows(c, d_rgsw, c->ws_io0.as<u32>(), (size_t)B * bits * 2 * ELL * 2 * K, s))) return rc;
      if ((rc = fold_rows(c, c->ws_io0.as<u32>(), c->ws_io0.as<u32>(), B, (int)(2 * bits), (size_t)bits * 2 * ELL * CT,
                          (size_t)ELL * CT, (size_t)bits * 2 * ELL * CT, (size_t)ELL * CT, s)))
        return rc;
    }
    u32* cur = c->ws_state0.as<u32>();
    u32* bufs[2] = {c->ws_ct0.as<u32>(), c->ws_ct1.as<u32>()};
    for (uint32_t j = 0; j < bits; ++j) {
      const int Cj = C >> j;
      RowsDesc r;
      r.lo = c->ws_io0.as<u32>() + (size_t)j * 2 * ELL * CT;
      r.lo_b = (size_t)bits * 2 * ELL * CT;
      r.hi = r.lo + (size_t)ELL * CT;
      r.hi_b = r.lo_b;
      r.slot = nullptr;
      u32* dst = bufs[j & 1];
      if ((rc = ext_product(c, cur, (size_t)Cj, B, Cj / 2, 1, dst, (size_t)Cj / 2, r,
                            xp_default((size_t)B * Cj / 2), s, &launches)))
        return rc;
      cur = dst;
    }
    return bitrev_rows(c, cur, d_out, (size_t)B * 2 * K, s);
  }

  // column-sharded worker step (cluster.answer_col_sharded): RowSel of all B
  // queries' row cts (brv, (B, d0)) against this shard's columns, then the
  // shard's log2(d1) ColTor stages with the given low-bit RGSW rows (natural,
  // (B, bits, 2 ELL)) -> one ct per query (natural).  Uses the capacity path's
  // column windows when the (B, d1) selection exceeds the budget.
  static int rowsel_coltor(gpir_ctx* c, gpir_db* db, const u32* d_rows, int B, const u32* d_rgsw, u32* d_out,
                           cudaStream_t s) {
    const uint32_t d1 = db->d1, bits = ilog2(d1);
    int rc;
    uint32_t launches = 0;
    if ((rc = c->ws_io0.ensure((size_t)B * std::max<uint32_t>(bits, 1) * 2 * ELL * CT * 4))) return rc;
    if (bits) {
      if ((rc = bitrev_rows(c, d_rgsw, c->ws_io0.as<u32>(), (size_t)B * bits * 2 * ELL * 2 * K, s))) return rc;
      if ((rc = fold_rows(c, c->ws_io0.as<u32>(), c->ws_io0.as<u32>(), B, (int)(2 * bits), (size_t)bits * 2 * ELL * CT,
                          (size_t)ELL * CT, (size_t)bits * 2 * ELL * CT, (size_t)ELL * CT, s)))
        return rc;
    }
    const RsPlan rp = rs_plan(c, B, db);
    const uint32_t wd = window_d1(c, B, db, rp), nw = d1 / wd, wbits = ilog2(wd);
    const size_t ctb = CT * 4;
    if ((rc = c->ws_sel.ensure(std::max(c->ws_sel.bytes, (size_t)B * wd * ctb)))) return rc;
    if ((rc = c->ws_ct0.ensure(std::max(c->ws_ct0.bytes, (size_t)B * std::max<uint32_t>(std::max(wd / 2, nw / 2), 1) * ctb))))
      return rc;
    if ((rc = c->ws_ct1.ensure(std::max(c->ws_ct1.bytes, (size_t)B * std::max<uint32_t>(std::max(wd / 4, nw / 4), 1) * ctb))))
      return rc;
    if ((rc = c->ws_part.ensure(std::max(c->ws_part.bytes, (size_t)B * nw * ctb)))) return rc;
    auto rows_of = [&](uint32_t j) {
      RowsDesc r;
      r.lo = c->ws_io0.as<u32>() + (size_t)j * 2 * ELL * CT;
      r.lo_b = (size_t)bits * 2 * ELL * CT;
      r.hi = r.lo + (size_t)ELL * CT;
      r.hi_b = r.lo_b;
      r.slot = nullptr;
      return r;
    };
    u32* bufs[2] = {c->ws_ct0.as<u32>(), c->ws_ct1.as<u32>()};
    u32* cur = nullptr;
    for (uint32_t w = 0; w < nw; ++w) {
      bool il = false;
      if ((rc = rowsel(c, d_rows, (size_t)db->d0 * CT, B, db, c->ws_sel.as<u32>(), s, &launches, nullptr, &rp, w > 0,
                       bits > 0, &il, nullptr, nw > 1 ? (int)(w * wd) : 0, nw > 1 ? (int)wd : 0)))
        return rc;
      cur = c->ws_sel.as<u32>();
      for (uint32_t j = 0; j < wbits; ++j) {
        const int C = (int)(wd >> j);
        const bool last = nw > 1 && j + 1 == wbits;
        u32* dst = last ? c->ws_part.as<u32>() + (size_t)w * CT : bufs[j & 1];
        if ((rc = ext_product(c, cur, (size_t)C, B, C / 2, (j == 0 && il) ? PAIRS_IL : 1, dst,
                              last ? (size_t)nw : (size_t)C / 2, rows_of(j), xp_default((size_t)B * C / 2), s,
                              &launches)))
          return rc;
        cur = dst;
      }
    }
    if (nw > 1) {
      cur = c->ws_part.as<u32>();
      for (uint32_t j = wbits; j < bits; ++j) {
        const int C = (int)(d1 >> j);
        u32* dst = bufs[j & 1];
        if ((rc = ext_product(c, cur, (size_t)C, B, C / 2, 1, dst, (size_t)C / 2, rows_of(j),
                              xp_default((size_t)B * C / 2), s, &launches)))
          return rc;
        cur = dst;
      }
    }
    return bitrev_rows(c, cur, d_out, (size_t)B * 2 * K, s);
  }

  // ---- operator-level parity entry points -------------------------------------------
  static int op_ntt(gpir_ctx* c, const u32* h_in, u32* h_out, uint32_t polys, int inverse);
  static int op_digits(gpir_ctx* c, const u32* h_coeff, int32_t* h_dig, uint32_t polys);
  static int op_expand_stage(gpir_ctx* c, const u32* h_state, int B, int C, const u32* h_ksk, int t, int mode,
                             u32* h_out);
  static int op_xp(gpir_ctx* c, const u32* h_cts, int B, int M, int pairs, const u32* h_rows, int mode, u32* h_out);
  static int op_rowsel(gpir_ctx* c, const u32* h_rows, int B, gpir_db* db, u32* h_out);
  // capacity mode: pack the byte planes in the k_rowsel_tk layout, release the u32 image
  static int db_compact(gpir_ctx* c, gpir_db* db) {
    if (db->compact) return 0;
    if (db->d0 > 256 || (K * N) % PK_P) FAIL(GPIR_UNSUPPORTED, "compact databases need d0 <= 256");
    db->compact = true;  // rs_plan: the TMEM-resident RowSel layout for every batch
    const RsPlan r = rs_plan(c, 128, db);
    db->compact = false;
    int rc;
    if (r.kind != 2) FAIL(GPIR_UNSUPPORTED, "compact databases need the tensor-core RowSel");
    if ((rc = ensure_d8(c, db, r, c->stream))) return rc;
    CK(cudaStreamSynchronize(c->stream));
    db->data.release();
    db->compact = true;
    return 0;
  }
  // client-side material (client.cuh)
  static int client_keygen(gpir_ctx* c, int slot, uint32_t stages, uint64_t seed, int8_t* h_secret);
  static int client_queries(gpir_ctx* c, const int8_t* h_secret, uint32_t plain_bits, uint32_t d0, uint32_t d1,
                            const uint32_t* istar, const uint32_t* jstar, uint32_t count, uint64_t seed, u32* h_out);
};

// plain NTT rows kernels for the parity entry point
template <int LOGN, int K>
__global__ void __launch_bounds__(NttCfg<LOGN>::T) k_ntt_rows(const u32* __restrict__ in, u32* __restrict__ out,
                                                             int inverse, Tables tb,
                                                             const __grid_constant__ TwConst tc) {
  constexpr int N = 1 << LOGN;
  __shared__ __align__(16) u32 xbuf[2 * N];
  NttState ns{xbuf, 0};
  const int row = blockIdx.x;
  const int i = row % K;
  const u32* src = in + (size_t)row * N;
  u32* dst = out + (size_t)row * N;
  if (inverse) {
    ntt_inv<LOGN>(
        ns, tb.inv + (size_t)i * N, tc.i[i], tb.mod[i], [&](int i0, u32(&x)[16]) { ld16(src + i0, x); },
        [&](int j, int, u32 v) { dst[j] = v; });
  } else {
    ntt_fwd<LOGN>(
        ns, tb.fwd + (size_t)i * N, tc.f[i], tb.mod[i], [&](int j) -> u32 { return __ldg(src + j); },
        [&](int i0, const u32(&x)[16]) { st16(dst + i0, x); });
  }
}

template <int LOGN, int K, int ELL>
int Engine<LOGN, K, ELL>::op_ntt(gpir_ctx* c, const u32* h_in, u32* h_out, uint32_t polys, int inverse) {
  const size_t rows = (size_t)polys * K, words = rows * N;
  int rc;
  if ((rc = c->ws_io0.ensure(words * 4)) || (rc = c->ws_io1.ensure(words * 4))) return rc;
  cudaStream_t s = c->stream;
  CK(cudaMemcpyAsync(c->ws_io0.p, h_in, words * 4, cudaMemcpyHostToDevice, s));
  if (inverse) {  // natural NTT values -> brv -> iNTT -> natural coefficients
    if ((rc = bitrev_rows(c, c->ws_io0.as<u32>(), c->ws_io1.as<u32>(), rows, s))) return rc;
    k_ntt_rows<LOGN, K><<<(unsigned)rows, T, 0, s>>>(c->ws_io1.as<u32>(), c->ws_io0.as<u32>(), 1, c->tb, c->tc);
    CKL();
    CK(cudaMemcpyAsync(h_out, c->ws_io0.p, words * 4, cudaMemcpyDeviceToHost, s));
  } else {
    k_ntt_rows<LOGN, K><<<(unsigned)rows, T, 0, s>>>(c->ws_io0.as<u32>(), c->ws_io1.as<u32>(), 0, c->tb, c->tc);
    CKL();
    if ((rc = bitrev_rows(c, c->ws_io1.as<u32>(), c->ws_io0.as<u32>(), rows, s))) return rc;
    CK(cudaMemcpyAsync(h_out, c->ws_io0.p, words * 4, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  return 0;
}

extern "C" {
static int install_keys_brv(gpir_ctx* c, int slot, const uint32_t* d_evks, uint32_t stages, const uint32_t* d_rgsw);
}

// z^i mod q_i for i < ell, [ell][K]
static std::vector<uint32_t> zpow_table(const gpir_ctx* c) {
  std::vector<uint32_t> z((size_t)c->ell * c->k);
  for (uint32_t i = 0; i < c->ell; ++i)
    for (uint32_t l = 0; l < c->k; ++l)
      z[(size_t)i * c->k + l] = (uint32_t)powmod(powmod(2, c->z_bits, c->q[l]), i, c->q[l]);
  return z;
}

template <int LOGN, int K, int ELL>
int Engine<LOGN, K, ELL>::client_keygen(gpir_ctx* c, int slot, uint32_t stages, uint64_t seed, int8_t* h_secret) {
  cudaStream_t s = c->stream;
  const size_t rows = (size_t)stages * ELL + 2 * ELL;
  DevBuf sc, snat, sbrv, zp, ph, ct;
  int rc;
  if ((rc = sc.ensure(N)) || (rc = snat.ensure((size_t)K * N * 4)) || (rc = sbrv.ensure((size_t)K * N * 4)) ||
      (rc = zp.ensure((size_t)ELL * K * 4)) || (rc = ph.ensure(rows * K * N * 4)) || (rc = ct.ensure(rows * CT * 4)))
    return rc;
  k_client_secret<<<(N + 255) / 256, 256, 0, s>>>(seed, N, K, sc.as<int8_t>(), snat.as<u32>(), c->tb);
  CKL();
  k_ntt_rows<LOGN, K><<<K, T, 0, s>>>(snat.as<u32>(), sbrv.as<u32>(), 0, c->tb, c->tc);
  CKL();
  const std::vector<uint32_t> z = zpow_table(c);
  CK(cudaMemcpyAsync(zp.p, z.data(), z.size() * 4, cudaMemcpyHostToDevice, s));
  const size_t tot = rows * K * N;
  k_client_key_phases<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(sbrv.as<u32>(), LOGN, K, (int)stages, ELL,
                                                                    zp.as<u32>(), ph.as<u32>(), c->tb);
  CKL();
  k_client_encrypt<LOGN, K><<<dim3((unsigned)rows, K), T, 0, s>>>(seed, 0, ph.as<u32>(), sbrv.as<u32>(), ct.as<u32>(),
                                                                 (int)c->error_bound, c->tb, c->tc);
  CKL();
  if ((rc = install_keys_brv(c, slot, ct.as<u32>(), stages, ct.as<u32>() + (size_t)stages * ELL * CT))) return rc;
  if (h_secret) CK(cudaMemcpy(h_secret, sc.p, N, cudaMemcpyDeviceToHost));
  return 0;
}

template <int LOGN, int K, int ELL>
int Engine<LOGN, K, ELL>::client_queries(gpir_ctx* c, const int8_t* h_secret, uint32_t plain_bits, uint32_t d0,
                                         uint32_t d1, const uint32_t* istar, const uint32_t* jstar, uint32_t count,
                                         uint64_t seed, u32* h_out) {
  cudaStream_t s = c->stream;
  const uint32_t total = leaves_of(d0, d1, ELL), stages = stages_of(total), bits = ilog2(d1);
  if (total > (uint32_t)N) FAIL(GPIR_INVALID_ARGUMENT, "expansion needs more slots than the ring has");
  if (!plain_bits || plain_bits > 32) FAIL(GPIR_INVALID_ARGUMENT, "plain modulus must be 2^1 .. 2^32");
  // payload (src/protocol.py:252-281): Delta / 2^stages at i*, z^dig / 2^stages at the column-bit slots
  u128 Q = 1;
  for (uint32_t l = 0; l < (uint32_t)K; ++l) Q *= c->q[l];
  const u128 delta = Q >> plain_bits;
  const std::vector<uint32_t> z = zpow_table(c);
  std::vector<uint32_t> pay((size_t)count * K * N, 0);
  for (uint32_t b = 0; b < count; ++b) {
    if (istar[b] >= d0 || jstar[b] >= d1) FAIL(GPIR_INVALID_ARGUMENT, "query index out of range");
    for (uint32_t l = 0; l < (uint32_t)K; ++l) {
      const uint64_t q = c->q[l];
      const uint64_t inv = powmod(powmod(2, stages, q), q - 2, q);
      uint32_t* row = pay.data() + ((size_t)b * K + l) * N;
      row[istar[b]] = (uint32_t)((uint64_t)(delta % q) * inv % q);
      for (uint32_t bit = 0; bit < bits; ++bit)
        if ((jstar[b] >> bit) & 1)
          for (uint32_t dg = 0; dg < (uint32_t)ELL; ++dg)
            row[d0 + bit * ELL + dg] = (uint32_t)((uint64_t)z[(size_t)dg * K + l] * inv % q);
    }
  }
  DevBuf sc, snat, sbrv, pnat, pbrv, ct, nat;
  int rc;
  const size_t pw = (size_t)count * K * N;
  if ((rc = sc.ensure(N)) || (rc = snat.ensure((size_t)K * N * 4)) || (rc = sbrv.ensure((size_t)K * N * 4)) ||
      (rc = pnat.ensure(pw * 4)) || (rc = pbrv.ensure(pw * 4)) || (rc = ct.ensure((size_t)count * CT * 4)) ||
      (rc = nat.ensure((size_t)count * CT * 4)))
    return rc;
  CK(cudaMemcpyAsync(sc.p, h_secret, N, cudaMemcpyHostToDevice, s));
  k_client_lift<<<(N + 255) / 256, 256, 0, s>>>(sc.as<int8_t>(), N, K, snat.as<u32>(), c->tb);
  CKL();
  k_ntt_rows<LOGN, K><<<K, T, 0, s>>>(snat.as<u32>(), sbrv.as<u32>(), 0, c->tb, c->tc);
  CKL();
  CK(cudaMemcpyAsync(pnat.p, pay.data(), pw * 4, cudaMemcpyHostToDevice, s));
  k_ntt_rows<LOGN, K><<<(unsigned)(count * K), T, 0, s>>>(pnat.as<u32>(), pbrv.as<u32>(), 0, c->tb, c->tc);
  CKL();
  k_client_encrypt<LOGN, K><<<dim3(count, K), T, 0, s>>>(seed, 1u << 20, pbrv.as<u32>(), sbrv.as<u32>(), ct.as<u32>(),
                                                        (int)c->error_bound, c->tb, c->tc);
  CKL();
  if ((rc = bitrev_rows(c, ct.as<u32>(), nat.as<u32>(), (size_t)count * 2 * K, s))) return rc;
  CK(cudaMemcpyAsync(h_out, nat.p, (size_t)count * CT * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

template <int LOGN, int K, int ELL>
int Engine<LOGN, K, ELL>::op_digits(gpir_ctx* c, const u32* h_coeff, int32_t* h_dig, uint32_t polys) {
  int rc;
  if ((rc = c->ws_io0.ensure((size_t)polys * K * N * 4)) || (rc = c->ws_io1.ensure((size_t)polys * ELL * N * 4)))
    return rc;
  cudaStream_t s = c->stream;
  CK(cudaMemcpyAsync(c->ws_io0.p, h_coeff, (size_t)polys * K * N * 4, cudaMemcpyHostToDevice, s));
  const size_t tot = (size_t)polys * N;
  k_op_dcp<LOGN, K, ELL><<<(unsigned)((tot / 4 + 255) / 256), 256, 0, s>>>(c->ws_io0.as<u32>(), (int)polys,
                                                                      c->ws_io1.as<int>(), c->tb, c->cc, ELL);
  CKL();
  CK(cudaMemcpyAsync(h_dig, c->ws_io1.p, (size_t)polys * ELL * N * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

template <int LOGN, int K, int ELL>
int Engine<LOGN, K, ELL>::op_expand_stage(gpir_ctx* c, const u32* h_state, int B, int C, const u32* h_ksk, int t,
                                          int mode, u32* h_out) {
  int rc;
  cudaStream_t s = c->stream;
  DevBuf st, ks, tmp, out;
  const size_t sw = (size_t)B * C * CT, kw = (size_t)B * ELL * CT, ow = (size_t)B * 2 * C * CT;
  if ((rc = st.ensure(sw * 4)) || (rc = ks.ensure(kw * 4)) || (rc = tmp.ensure(std::max(sw, kw) * 4)) ||
      (rc = out.ensure(ow * 4)))
    return rc;
  CK(cudaMemcpyAsync(tmp.p, h_state, sw * 4, cudaMemcpyHostToDevice, s));
  if ((rc = bitrev_rows(c, tmp.as<u32>(), st.as<u32>(), sw >> LOGN, s))) return rc;
  CK(cudaMemcpyAsync(tmp.p, h_ksk, kw * 4, cudaMemcpyHostToDevice, s));
  if ((rc = bitrev_rows(c, tmp.as<u32>(), ks.as<u32>(), kw >> LOGN, s))) return rc;
  if ((rc = fold_rows(c, ks.as<u32>(), ks.as<u32>(), B, 1, (size_t)ELL * CT, 0, (size_t)ELL * CT, 0, s))) return rc;
  RowsDesc r;
  r.lo = ks.as<u32>();
  r.lo_b = (size_t)ELL * CT;
  r.hi = r.lo;
  r.hi_b = r.lo_b;
  r.slot = nullptr;
  uint32_t launches = 0;
  if ((rc = expand_stage(c, st.as<u32>(), B, C, out.as<u32>(), 2 * C, t, r, mode, s, &launches))) return rc;
  if ((rc = tmp.ensure(ow * 4))) return rc;
  if ((rc = bitrev_rows(c, out.as<u32>(), tmp.as<u32>(), ow >> LOGN, s))) return rc;
  CK(cudaMemcpyAsync(h_out, tmp.p, ow * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  st.release();
  ks.release();
  tmp.release();
  out.release();
  return 0;
}

template <int LOGN, int K, int ELL>
int Engine<LOGN, K, ELL>::op_xp(gpir_ctx* c, const u32* h_cts, int B, int M, int pairs, const u32* h_rows, int mode,
                                u32* h_out) {
  int rc;
  cudaStream_t s = c->stream;
  const int Min = pairs ? 2 * M : M;
  DevBuf in, rw, tmp, out;
  const size_t iw = (size_t)B * Min * CT, rwn = (size_t)B * 2 * ELL * CT, ow = (size_t)B * M * CT;
  if ((rc = in.ensure(iw * 4)) || (rc = rw.ensure(rwn * 4)) || (rc = tmp.ensure(std::max(iw, rwn) * 4)) ||
      (rc = out.ensure(ow * 4)))
    return rc;
  CK(cudaMemcpyAsync(tmp.p, h_cts, iw * 4, cudaMemcpyHostToDevice, s));
  if ((rc = bitrev_rows(c, tmp.as<u32>(), in.as<u32>(), iw >> LOGN, s))) return rc;
  CK(cudaMemcpyAsync(tmp.p, h_rows, rwn * 4, cudaMemcpyHostToDevice, s));
  if ((rc = bitrev_rows(c, tmp.as<u32>(), rw.as<u32>(), rwn >> LOGN, s))) return rc;
  if ((rc = fold_rows(c, rw.as<u32>(), rw.as<u32>(), B, 2, 2 * (size_t)ELL * CT, (size_t)ELL * CT,
                      2 * (size_t)ELL * CT, (size_t)ELL * CT, s)))
    return rc;
  RowsDesc r;
  r.lo = rw.as<u32>();
  r.lo_b = 2 * (size_t)ELL * CT;
  r.hi = r.lo + (size_t)ELL * CT;
  r.hi_b = r.lo_b;
  r.slot = nullptr;
  uint32_t launches = 0;
  if ((rc = ext_product(c, in.as<u32>(), (size_t)Min, B, M, pairs, out.as<u32>(), (size_t)M, r, mode, s, &launches)))
    return rc;
  if ((rc = bitrev_rows(c, out.as<u32>(), tmp.as<u32>(), ow >> LOGN, s))) return rc;
  CK(cudaMemcpyAsync(h_out, tmp.p, ow * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  in.release();
  rw.release();
  tmp.release();
  out.release();
  return 0;
}

template <int LOGN, int K, int ELL>
int Engine<LOGN, K, ELL>::op_rowsel(gpir_ctx* c, const u32* h_rows, int B, gpir_db* db, u32* h_out) {
  int rc;
  cudaStream_t s = c->stream;
  DevBuf in, tmp, out;
  const size_t iw = (size_t)B * db->d0 * CT, ow = (size_t)B * db->d1 * CT;
  if ((rc = in.ensure(iw * 4)) || (rc = tmp.ensure(std::max(iw, ow) * 4)) || (rc = out.ensure(ow * 4))) return rc;
  CK(cudaMemcpyAsync(tmp.p, h_rows, iw * 4, cudaMemcpyHostToDevice, s));
  if ((rc = bitrev_rows(c, tmp.as<u32>(), in.as<u32>(), iw >> LOGN, s))) return rc;
  uint32_t launches = 0;
  if ((rc = rowsel(c, in.as<u32>(), (size_t)db->d0 * CT, B, db, out.as<u32>(), s, &launches))) return rc;
  if ((rc = bitrev_rows(c, out.as<u32>(), tmp.as<u32>(), ow >> LOGN, s))) return rc;
  CK(cudaMemcpyAsync(h_out, tmp.p, ow * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  in.release();
  tmp.release();
  out.release();
  return 0;
}

// DB encode launcher
template <int LOGN, int K>
static int db_encode_launch(gpir_ctx* c, const uint8_t* d_recs, int rec_bytes, int d0, int d1, int plain_bits,
                            u32* db, cudaStream_t s) {
  k_db_encode<LOGN, K><<<dim3(d0 * d1, K), NttCfg<LOGN>::T, 0, s>>>(d_recs, rec_bytes, d0, d1, plain_bits, db, c->tb, c->tc);
  CKL();
  return 0;
}

#include "wire_codec.h"

// ---------------------------------------------------------------------------
// dispatch over compiled (LOGN, K, ELL) combinations

#define GPIR_COMBOS(X) \
  X(12, 4, 5)          \
  X(8, 2, 5)           \
  X(6, 2, 6)

extern "C" {

const char* gpir_last_error(void) { return g_err.c_str(); }
const char* gpir_version(void) { return "gpir-b200 0.1 (sm_100a)"; }

int gpir_supported(uint32_t n, uint32_t k, uint32_t ell) {
  const uint32_t logn = ilog2(n);
  if ((1u << logn) != n) return 0;
  const uint32_t key = logn * 10000 + k * 100 + ell;
#define SUP(L, K_, E) \
  if (key == L * 10000 + K_ * 100 + E) return 1;
  GPIR_COMBOS(SUP)
#undef SUP
  return 0;
}

gpir_ctx* gpir_ctx_create(int device, uint32_t n, uint32_t k, const uint32_t* q, const uint32_t* psi, uint32_t z_bits,
                          uint32_t ell) {
  if (!gpir_supported(n, k, ell)) {
    g_err = "unsupported ring/gadget (n=" + std::to_string(n) + ", k=" + std::to_string(k) +
            ", ell=" + std::to_string(ell) + ") for this build";
    return nullptr;
  }
  if (z_bits < 2 || z_bits > 31 || k > kMaxLimbs || ell > kMaxEll) {
    g_err = "invalid gadget parameters";
    return nullptr;
  }
  u128 Q = 1;
  const uint32_t logn_ = ilog2(n);
  for (uint32_t i = 0; i < k; ++i) {
    // lazy forward transform bound (values < (2 log2 n + 1) q), as src/ring.py:208-210
    if ((uint64_t)q[i] * (2 * logn_ + 1) >= (1ull << 32)) {
      g_err = "prime too large for the lazy 32-bit transform: q * (2 log2 n + 1) must be < 2^32";
      return nullptr;
    }
    Q *= q[i];
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    g_err = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
    return nullptr;
  }
  gpir_ctx* c = new gpir_ctx();
  c->device = device;
  c->n = n;
  c->logn = ilog2(n);
  c->k = k;
  c->ell = ell;
  c->z_bits = z_bits;
  c->q.assign(q, q + k);
  c->psi.assign(psi, psi + k);
  if (build_tables(c)) {
    delete c;
    return nullptr;
  }
  cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (const char* ge = getenv("GPIR_GRAPH")) c->use_graph = atoi(ge);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  for (auto& ev : c->ev) cudaEventCreate(&ev);
  cudaEventCreateWithFlags(&c->ev_legacy, cudaEventDisableTiming);
  return c;
}

void gpir_ctx_destroy(gpir_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (DevBuf* b : {&c->tw_fwd, &c->tw_inv, &c->mono, &c->evk_pool, &c->rgsw_pool, &c->ws_state0, &c->ws_state1,
                    &c->ws_arows, &c->ws_sel, &c->ws_y, &c->ws_part, &c->ws_ct0, &c->ws_ct1, &c->ws_kslot, &c->ws_coeff, &c->ws_dig,
                    &c->ws_dn, &c->ws_io0, &c->ws_io1, &c->ws_a8})
    b->release();
  for (auto& ev : c->ev) cudaEventDestroy(ev);
  for (auto& ev : c->evp) cudaEventDestroy(ev);
  if (c->ev_legacy) cudaEventDestroy(c->ev_legacy);
  for (auto& g : c->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  cudaStreamDestroy(c->stream);
  delete c;
}

int gpir_ctx_device(const gpir_ctx* c) { return c ? c->device : -1; }

uint64_t gpir_launch_count(void) { return g_launches.load(); }

int gpir_set_graphs(gpir_ctx* c, int on) {
  if (!c) FAIL(GPIR_INVALID_ARGUMENT, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  c->use_graph = on ? 1 : 0;
  return 0;
}

int gpir_set_capacity(gpir_ctx* c, uint64_t sel_budget_bytes, uint32_t max_batch) {
  if (!c) FAIL(GPIR_INVALID_ARGUMENT, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  c->sel_budget = (size_t)sel_budget_bytes;
  c->max_batch = (int)max_batch;
  return 0;
}

int gpir_set_rowsel_engine(gpir_ctx* c, int engine) {
  if (!c || engine < 0 || engine > 2) FAIL(GPIR_INVALID_ARGUMENT, "engine must be 0 (auto), 1 (CUDA cores) or 2 (tensor cores)");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  c->rowsel_engine = engine;
  return 0;
}

static gpir_db* db_encode_impl(gpir_ctx* c, const uint8_t* records, bool on_device, uint32_t d0, uint32_t d1,
                               uint32_t record_bytes, uint32_t plain_bits) {
  if (!c || !records || !d0 || !d1 || (d1 & (d1 - 1))) {
    g_err = "invalid database geometry";
    return nullptr;
  }
  if (plain_bits % 8 || plain_bits == 0 || plain_bits > 32 || (uint64_t)record_bytes * 8 > (uint64_t)c->n * plain_bits) {
    g_err = "record does not fit one plaintext polynomial";
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  cudaSetDevice(c->device);
  gpir_db* db = new gpir_db();
  db->d0 = d0;
  db->d1 = d1;
  const size_t recs = (size_t)d0 * d1;
  DevBuf raw;
  int rc = on_device ? 0 : raw.ensure(std::max<size_t>(recs * record_bytes, 16));
  if (!rc) rc = db->data.ensure(recs * c->k * c->n * 4);
  if (!rc && !on_device &&
      cudaMemcpyAsync(raw.p, records, recs * record_bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
    rc = GPIR_CUDA_ERROR, g_err = "db upload failed";
  const uint8_t* src = on_device ? records : raw.as<uint8_t>();
  if (!rc) {
    switch (c->logn * 100 + c->k) {
#define ENC(L, K_, E) \
  case L * 100 + K_: rc = db_encode_launch<L, K_>(c, src, (int)record_bytes, (int)d0, (int)d1, (int)plain_bits, db->data.as<u32>(), c->stream); break;
      GPIR_COMBOS(ENC)
#undef ENC
      default:
        rc = GPIR_UNSUPPORTED;
    }
  }
  if (!rc && cudaStreamSynchronize(c->stream) != cudaSuccess) rc = GPIR_CUDA_ERROR, g_err = "db encode failed";
  raw.release();
  if (rc) {
    db->data.release();
    delete db;
    return nullptr;
  }
  return db;
}

gpir_db* gpir_db_encode(gpir_ctx* c, const uint8_t* records, uint32_t d0, uint32_t d1, uint32_t record_bytes,
                        uint32_t plain_bits) {
  return db_encode_impl(c, records, false, d0, d1, record_bytes, plain_bits);
}

gpir_db* gpir_db_encode_dev(gpir_ctx* c, const uint8_t* d_records, uint32_t d0, uint32_t d1, uint32_t record_bytes,
                            uint32_t plain_bits) {
  return db_encode_impl(c, d_records, true, d0, d1, record_bytes, plain_bits);
}

gpir_db* gpir_db_upload(gpir_ctx* c, const uint32_t* pmajor, uint32_t d0, uint32_t d1) {
  if (!c || !pmajor || !d0 || !d1 || (d1 & (d1 - 1))) {
    g_err = "invalid database geometry";
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  cudaSetDevice(c->device);
  gpir_db* db = new gpir_db();
  db->d0 = d0;
  db->d1 = d1;
  const size_t words = (size_t)d0 * d1 * c->k * c->n;
  DevBuf tmp;
  int rc = tmp.ensure(words * 4);
  if (!rc) rc = db->data.ensure(words * 4);
  if (!rc && cudaMemcpyAsync(tmp.p, pmajor, words * 4, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
    rc = GPIR_CUDA_ERROR, g_err = "db upload failed";
  if (!rc) rc = bitrev_rows(c, tmp.as<u32>(), db->data.as<u32>(), words >> c->logn, c->stream);
  if (!rc && cudaStreamSynchronize(c->stream) != cudaSuccess) rc = GPIR_CUDA_ERROR, g_err = "db upload failed";
  tmp.release();
  if (rc) {
    db->data.release();
    delete db;
    return nullptr;
  }
  return db;
}

// ---- GPDB container (save_database / load_database, src/wire.py:365-410) ----
// Header "<4sHIIIIBBB": magic, version, d0, d1, record_bytes, n, k, plain_bits,
// layout (0 P-major (d1, d0, p), 1 transposed (p, d1, d0)); k u64 primes; the
// <u4 payload.  The payload streams through a pinned 64 MiB staging buffer into
// device memory; a transposed image is transposed on the GPU.
static const size_t kDbHead = 25;

gpir_db* gpir_db_load(gpir_ctx* c, const char* path, uint32_t expect_plain_bits, uint32_t* d0_out, uint32_t* d1_out,
                      uint32_t* record_bytes_out, uint32_t* plain_bits_out) {
  using namespace gpir_wire;
  g_off = -1;  // set >= 0 only by a parse error
  if (!c || !path) {
    g_err = "invalid argument";
    return nullptr;
  }
  FILE* fh = fopen(path, "rb");
  if (!fh) {
    g_err = std::string("cannot open ") + path;
    return nullptr;
  }
  struct Closer {
    FILE* f;
    ~Closer() { fclose(f); }
  } closer{fh};
  uint8_t head[kDbHead];
  const size_t got = fread(head, 1, kDbHead, fh);
  auto fail = [&](const std::string& m, int64_t off) -> gpir_db* {
    parse_fail(m, off);
    return nullptr;
  };
  if (got < kDbHead) return fail("truncated database header", (int64_t)got);
  if (memcmp(head, kDbMagic, 4) != 0) {
    char m[64];
    snprintf(m, sizeof m, "bad database magic b'%c%c%c%c'", head[0], head[1], head[2], head[3]);
    return fail(m, 0);
  }
  const uint16_t ver = rd<uint16_t>(head + 4);
  if (ver != kVersion) return fail("unsupported database version " + std::to_string(ver), 4);
  const uint32_t d0 = rd<uint32_t>(head + 6), d1 = rd<uint32_t>(head + 10), rb = rd<uint32_t>(head + 14);
  const uint32_t n = rd<uint32_t>(head + 18), k = head[22], pb = head[23], layout = head[24];
  std::vector<uint64_t> qs(k);
  if (k && fread(qs.data(), 8, k, fh) != k) return fail("truncated database header", (int64_t)kDbHead);
  bool match = n == c->n && k == c->k && (!expect_plain_bits || expect_plain_bits == pb);
  for (uint32_t i = 0; match && i < k; ++i) match = qs[i] == c->q[i];
  if (!match) return fail("database parameters do not match the supplied profile", (int64_t)kDbHead);
  if (!d0 || !d1 || (d1 & (d1 - 1)) || layout > 1) return fail("bad database geometry", 6);
  const size_t words = (size_t)d0 * d1 * k * n;
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  cudaSetDevice(c->device);
  gpir_db* db = new gpir_db();
  db->d0 = d0;
  db->d1 = d1;
  DevBuf tmp, tr;
  void* pinned = nullptr;
  const size_t chunk = (size_t)64 << 20;
  int rc = tmp.ensure(words * 4);
  if (!rc) rc = db->data.ensure(words * 4);
  if (!rc && cudaMallocHost(&pinned, chunk) != cudaSuccess) rc = GPIR_CUDA_ERROR, g_err = "pinned staging";
  size_t done = 0;
  while (!rc && done < words * 4) {
    const size_t want = std::min(chunk, words * 4 - done);
    const size_t r = fread(pinned, 1, want, fh);
    if (r < want) {
      parse_fail("truncated database payload", (int64_t)(kDbHead + done + r));
      rc = -6;
      break;
    }
    if (cudaMemcpy(tmp.as<uint8_t>() + done, pinned, want, cudaMemcpyHostToDevice) != cudaSuccess)
      rc = GPIR_CUDA_ERROR, g_err = "db upload failed";
    done += want;
  }
  const u32* pm = tmp.as<u32>();
  if (!rc && layout == 1) {  // (p, d1, d0) -> (d1, d0, p)
    rc = tr.ensure(words * 4);
    if (!rc) {
      const size_t P = (size_t)k * n, R = (size_t)d1 * d0;
      dim3 g((unsigned)((R + 31) / 32), (unsigned)((P + 31) / 32));
      k_transpose32<<<g, dim3(32, 8), 0, c->stream>>>(tmp.as<u32>(), tr.as<u32>(), P, R);
      if (cudaGetLastError() != cudaSuccess) rc = GPIR_CUDA_ERROR, g_err = "transpose launch";
      pm = tr.as<u32>();
    }
  }
  if (!rc) rc = bitrev_rows(c, pm, db->data.as<u32>(), words >> c->logn, c->stream);
  if (!rc && cudaStreamSynchronize(c->stream) != cudaSuccess) rc = GPIR_CUDA_ERROR, g_err = "db load failed";
  if (pinned) cudaFreeHost(pinned);
  tmp.release();
  tr.release();
  if (rc) {
    db->data.release();
    delete db;
    return nullptr;
  }
  if (d0_out) *d0_out = d0;
  if (d1_out) *d1_out = d1;
  if (record_bytes_out) *record_bytes_out = rb;
  if (plain_bits_out) *plain_bits_out = pb;
  return db;
}

int gpir_db_save(gpir_ctx* c, const gpir_db* db, const char* path, uint32_t record_bytes, uint32_t plain_bits) {
  using namespace gpir_wire;
  if (!c || !db || !path) FAIL(GPIR_INVALID_ARGUMENT, "invalid argument");
  const size_t words = (size_t)db->d0 * db->d1 * c->k * c->n;
  std::vector<uint32_t> host(words);
  int rc = gpir_db_download(c, db, host.data());
  if (rc) return rc;
  FILE* fh = fopen(path, "wb");
  if (!fh) FAIL(GPIR_INVALID_ARGUMENT, std::string("cannot open ") + path);
  uint8_t head[kDbHead];
  memcpy(head, kDbMagic, 4);
  wr<uint16_t>(head + 4, kVersion);
  wr<uint32_t>(head + 6, db->d0);
  wr<uint32_t>(head + 10, db->d1);
  wr<uint32_t>(head + 14, record_bytes);
  wr<uint32_t>(head + 18, c->n);
  head[22] = (uint8_t)c->k;
  head[23] = (uint8_t)plain_bits;
  head[24] = 0;  // P-major
  bool ok = fwrite(head, 1, kDbHead, fh) == kDbHead;
  for (uint32_t i = 0; ok && i < c->k; ++i) {
    const uint64_t q = c->q[i];
    ok = fwrite(&q, 8, 1, fh) == 1;
  }
  ok = ok && fwrite(host.data(), 4, words, fh) == words;
  ok = (fclose(fh) == 0) && ok;
  if (!ok) FAIL(GPIR_INVALID_ARGUMENT, std::string("write failed: ") + path);
  return 0;
}

int gpir_db_compact(gpir_ctx* c, gpir_db* db) {
  if (!c || !db) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  switch (c->logn * 10000 + c->k * 100 + c->ell) {
    case 120405: return Engine<12, 4, 5>::db_compact(c, db);
    case 80205: return Engine<8, 2, 5>::db_compact(c, db);
    case 60206: return Engine<6, 2, 6>::db_compact(c, db);
    default: FAIL(GPIR_UNSUPPORTED, "unsupported combination");
  }
}

int gpir_db_download(gpir_ctx* c, const gpir_db* db, uint32_t* out) {
  if (!c || !db || !out) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  if (db->compact) FAIL(GPIR_INVALID_STATE, "compact database: only the byte-plane image is resident");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  const size_t words = (size_t)db->d0 * db->d1 * c->k * c->n;
  DevBuf tmp;
  int rc = tmp.ensure(words * 4);
  if (rc) return rc;
  if ((rc = bitrev_rows(c, db->data.as<u32>(), tmp.as<u32>(), words >> c->logn, c->stream))) return rc;
  CK(cudaMemcpyAsync(out, tmp.p, words * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  tmp.release();
  return 0;
}

void gpir_db_destroy(gpir_ctx* c, gpir_db* db) {
  if (!db) return;
  if (c) {
    std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    db->data.release();
    db->d8.release();
  }
  delete db;
}

size_t gpir_db_bytes(const gpir_db* db) { return db ? db->data.bytes + db->d8.bytes : 0; }

// grow the key pools (slots x max stages), preserving existing keys; caller holds c->mu
static int ensure_key_pool(gpir_ctx* c, int slot, uint32_t stages) {
  const size_t CT = c->ct_words();
  const size_t ell = c->ell;
  int rc;
  const uint32_t want_slots = std::max<uint32_t>(c->key_slots, (uint32_t)slot + 1);
  const uint32_t want_stages = std::max<uint32_t>(c->key_stages, std::max<uint32_t>(stages, 1));
  if (want_slots == c->key_slots && want_stages == c->key_stages) return 0;
  const uint32_t ns = std::max<uint32_t>(want_slots, c->key_slots ? 2 * c->key_slots : 4);
  DevBuf ne, nr;
  if ((rc = ne.ensure((size_t)ns * want_stages * ell * CT * 4))) return rc;
  if ((rc = nr.ensure((size_t)ns * 2 * ell * CT * 4))) return rc;
  for (uint32_t sl = 0; sl < c->key_slots; ++sl) {
    if (c->slot_stages[sl] > 0)
      CK(cudaMemcpyAsync(ne.as<u32>() + (size_t)sl * want_stages * ell * CT,
                         c->evk_pool.as<u32>() + (size_t)sl * c->key_stages * ell * CT,
                         (size_t)c->slot_stages[sl] * ell * CT * 4, cudaMemcpyDeviceToDevice, c->stream));
    if (c->slot_rgsw[sl])
      CK(cudaMemcpyAsync(nr.as<u32>() + (size_t)sl * 2 * ell * CT, c->rgsw_pool.as<u32>() + (size_t)sl * 2 * ell * CT,
                         2 * ell * CT * 4, cudaMemcpyDeviceToDevice, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  c->evk_pool.release();
  c->rgsw_pool.release();
  c->evk_pool = ne;
  c->rgsw_pool = nr;
  ne.p = nullptr;
  nr.p = nullptr;
  c->slot_stages.resize(ns, -1);
  c->slot_rgsw.resize(ns, 0);
  c->key_slots = ns;
  c->key_stages = want_stages;
  return 0;
}

// install device key rows in internal (brv) order into slot: fold into the pool
static int install_keys_brv(gpir_ctx* c, int slot, const uint32_t* d_evks, uint32_t stages, const uint32_t* d_rgsw) {
  const size_t CT = c->ct_words(), ell = c->ell;
  int rc;
  if ((rc = ensure_key_pool(c, slot, stages))) return rc;
  if (stages) {
    u32* dst = c->evk_pool.as<u32>() + (size_t)slot * c->key_stages * ell * CT;
    if ((rc = fold_rows(c, d_evks, dst, 1, (int)stages, 0, ell * CT, 0, ell * CT, c->stream))) return rc;
  }
  c->slot_rgsw[slot] = 0;
  if (d_rgsw) {
    u32* dst = c->rgsw_pool.as<u32>() + (size_t)slot * 2 * ell * CT;
    if ((rc = fold_rows(c, d_rgsw, dst, 1, 2, 0, ell * CT, 0, ell * CT, c->stream))) return rc;
    c->slot_rgsw[slot] = 1;
  }
  CK(cudaStreamSynchronize(c->stream));
  c->slot_stages[slot] = (int)stages;
  return 0;
}

int gpir_keys_put(gpir_ctx* c, int slot, const uint32_t* evks, uint32_t stages, const uint32_t* sk_rgsw) {
  if (!c || slot < 0 || (stages && !evks)) FAIL(GPIR_INVALID_ARGUMENT, "invalid key upload");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  const size_t CT = c->ct_words();
  const size_t ell = c->ell;
  int rc;
  const size_t ew = (size_t)stages * ell * CT, rw = 2 * ell * CT;
  DevBuf tmp, brv;
  if ((rc = tmp.ensure(std::max<size_t>(ew + rw, 1) * 4)) || (rc = brv.ensure(std::max<size_t>(ew + rw, 1) * 4)))
    return rc;
  if (stages) {
    CK(cudaMemcpyAsync(tmp.p, evks, ew * 4, cudaMemcpyHostToDevice, c->stream));
    if ((rc = bitrev_rows(c, tmp.as<u32>(), brv.as<u32>(), ew >> c->logn, c->stream))) return rc;
  }
  if (sk_rgsw) {
    CK(cudaMemcpyAsync(tmp.as<u32>() + ew, sk_rgsw, rw * 4, cudaMemcpyHostToDevice, c->stream));
    if ((rc = bitrev_rows(c, tmp.as<u32>() + ew, brv.as<u32>() + ew, rw >> c->logn, c->stream))) return rc;
  }
  rc = install_keys_brv(c, slot, brv.as<u32>(), stages, sk_rgsw ? brv.as<u32>() + ew : nullptr);
  tmp.release();
  brv.release();
  return rc;
}

#define DISPATCH_CASE_CKG(L, K_, E) \
  case L * 10000 + K_ * 100 + E:    \
    return Engine<L, K_, E>::client_keygen(c, slot, stages, seed, secret_out);

int gpir_client_keygen(gpir_ctx* c, int slot, uint32_t stages, uint64_t seed, uint32_t error_bound,
                       int8_t* secret_out) {
  if (!c || slot < 0 || stages > 31) FAIL(GPIR_INVALID_ARGUMENT, "invalid client keygen request");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  c->error_bound = error_bound;
  switch (c->logn * 10000 + c->k * 100 + c->ell) {
    GPIR_COMBOS(DISPATCH_CASE_CKG)
    default:
      FAIL(GPIR_UNSUPPORTED, "unsupported combination");
  }
}

#define DISPATCH_CASE_CQ(L, K_, E) \
  case L * 10000 + K_ * 100 + E:   \
    return Engine<L, K_, E>::client_queries(c, secret, plain_bits, d0, d1, i_star, j_star, count, seed, queries_out);

int gpir_client_queries(gpir_ctx* c, const int8_t* secret, uint32_t plain_bits, uint32_t error_bound, uint32_t d0,
                        uint32_t d1, const uint32_t* i_star, const uint32_t* j_star, uint32_t count, uint64_t seed,
                        uint32_t* queries_out) {
  if (!c || !secret || !i_star || !j_star || !queries_out || !d0 || !d1 || (d1 & (d1 - 1)))
    FAIL(GPIR_INVALID_ARGUMENT, "invalid client query request");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  c->error_bound = error_bound;
  if (!count) return 0;
  switch (c->logn * 10000 + c->k * 100 + c->ell) {
    GPIR_COMBOS(DISPATCH_CASE_CQ)
    default:
      FAIL(GPIR_UNSUPPORTED, "unsupported combination");
  }
}

int gpir_keys_drop(gpir_ctx* c, int slot) {
  if (!c) FAIL(GPIR_INVALID_ARGUMENT, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  if (slot >= 0 && (uint32_t)slot < c->key_slots) {
    c->slot_stages[slot] = -1;
    c->slot_rgsw[slot] = 0;
  }
  return 0;
}

#define DISPATCH_CASE_ANSWER(L, K_, E) \
  case L * 10000 + K_ * 100 + E:       \
    return Engine<L, K_, E>::answer_dev(c, const_cast<gpir_db*>(db), d_q, key_slots, (int)B, eq_modes, n_eq, ct_modes, n_ct, d_out, s, stats);

static int answer_dev_dispatch(gpir_ctx* c, const gpir_db* db, const uint32_t* d_q, const int32_t* key_slots,
                               uint32_t B, const uint8_t* eq_modes, uint32_t n_eq, const uint8_t* ct_modes,
                               uint32_t n_ct, uint32_t* d_out, cudaStream_t s, gpir_stats* stats) {
  switch (c->logn * 10000 + c->k * 100 + c->ell) {
    GPIR_COMBOS(DISPATCH_CASE_ANSWER)
    default:
      FAIL(GPIR_UNSUPPORTED, "unsupported combination");
  }
}

int gpir_answer_batch_dev(gpir_ctx* c, const gpir_db* db, const uint32_t* d_queries, const int32_t* key_slots,
                          uint32_t B, const uint8_t* eq_modes, uint32_t n_eq, const uint8_t* ct_modes, uint32_t n_ct,
                          uint32_t* d_responses, void* stream, gpir_stats* stats) {
  if (!c || !db || !d_queries || !key_slots || !d_responses) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  if (B == 0) return 0;
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  cudaStream_t s = pick_stream(c, stream);
  if (stats) memset(stats, 0, sizeof(*stats));
  int rc = answer_dev_dispatch(c, db, d_queries, key_slots, B, eq_modes, n_eq, ct_modes, n_ct, d_responses, s, stats);
  if (rc) return rc;
  if (!stream) CK(cudaStreamSynchronize(s));
  return 0;
}

int gpir_answer_batch(gpir_ctx* c, const gpir_db* db, const uint32_t* queries, const int32_t* key_slots, uint32_t B,
                      const uint8_t* eq_modes, uint32_t n_eq, const uint8_t* ct_modes, uint32_t n_ct,
                      uint32_t* responses_out, gpir_stats* stats) {
  if (!c || !db || !queries || !key_slots || !responses_out) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  if (B == 0) return 0;
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const size_t words = (size_t)B * c->ct_words();
  int rc;
  if ((rc = c->ws_io0.ensure(words * 4)) || (rc = c->ws_io1.ensure(words * 4))) return rc;
  if (stats) memset(stats, 0, sizeof(*stats));
  CK(cudaEventRecord(c->ev[7], s));
  CK(cudaMemcpyAsync(c->ws_io0.p, queries, words * 4, cudaMemcpyHostToDevice, s));
  CK(cudaEventRecord(c->ev[8], s));
  rc = answer_dev_dispatch(c, db, c->ws_io0.as<u32>(), key_slots, B, eq_modes, n_eq, ct_modes, n_ct,
                           c->ws_io1.as<u32>(), s, stats);
  if (rc) return rc;
  CK(cudaEventRecord(c->ev[9], s));
  CK(cudaMemcpyAsync(responses_out, c->ws_io1.p, words * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaEventRecord(c->ev[10], s));
  CK(cudaEventSynchronize(c->ev[10]));
  if (stats) {
    cudaEventElapsedTime(&stats->ms_h2d, c->ev[7], c->ev[8]);
    cudaEventElapsedTime(&stats->ms_d2h, c->ev[9], c->ev[10]);
  }
  return 0;
}

int gpir_set_stage_timing(gpir_ctx* c, int on) {
  if (!c) FAIL(GPIR_INVALID_ARGUMENT, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  c->stage_timing = on ? 1 : 0;
  return 0;
}

int gpir_stage_times(gpir_ctx* c, gpir_stage_time* out, uint32_t cap) {
  if (!c) FAIL(GPIR_INVALID_ARGUMENT, "null context");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  const uint32_t m = std::min<uint32_t>(cap, (uint32_t)c->last_stages.size());
  for (uint32_t i = 0; i < m && out; ++i) out[i] = c->last_stages[i];
  return (int)c->last_stages.size();
}

int gpir_plan(gpir_ctx* c, uint32_t d0, uint32_t d1, uint32_t B, uint8_t* eq_modes, uint32_t n_eq, uint8_t* ct_modes,
              uint32_t n_ct) {
  if (!c) FAIL(GPIR_INVALID_ARGUMENT, "null context");
  const uint32_t total = leaves_of(d0, d1, c->ell);
  const uint32_t st = stages_of(total), bits = ilog2(d1);
  for (uint32_t t = 0; t < n_eq && t < st; ++t)
    eq_modes[t] = (size_t)B * std::min<uint32_t>(1u << t, total) >= kEqStageNodes ? 3 : 0;
  for (uint32_t j = 0; j < n_ct && j < bits; ++j) ct_modes[j] = (size_t)B * (d1 >> (j + 1)) >= kXpStageCts ? 3 : 0;
  return 0;
}

#define DISPATCH_CASE_SHARD(L, K_, E) \
  case L * 10000 + K_ * 100 + E:      \
    rc = Engine<L, K_, E>::shard_answer(c, const_cast<gpir_db*>(db), d1_total, d_queries, key_slots, (int)B, d_partials, d_high_rgsw, s, stats); break;

int gpir_shard_answer(gpir_ctx* c, const gpir_db* db, uint32_t d1_total, const uint32_t* d_queries,
                      const int32_t* key_slots, uint32_t B, uint32_t* d_partials, uint32_t* d_high_rgsw, void* stream,
                      gpir_stats* stats) {
  if (!c || !db || !d_queries || !key_slots || !d_partials) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  cudaStream_t s = pick_stream(c, stream);
  if (stats) memset(stats, 0, sizeof(*stats));
  int rc;
  switch (c->logn * 10000 + c->k * 100 + c->ell) {
    GPIR_COMBOS(DISPATCH_CASE_SHARD)
    default:
      FAIL(GPIR_UNSUPPORTED, "unsupported combination");
  }
  if (rc) return rc;
  if (!stream) CK(cudaStreamSynchronize(s));
  return 0;
}

#define DISPATCH_CASE_SHX(L, K_, E) \
  case L * 10000 + K_ * 100 + E:    \
    rc = Engine<L, K_, E>::sh_expand(c, d0, d1, d_queries, key_slots, (int)B, d_rows, s); break;

int gpir_sharded_expand(gpir_ctx* c, uint32_t d0, uint32_t d1, const uint32_t* d_queries, const int32_t* key_slots,
                        uint32_t B, uint32_t* d_rows, void* stream) {
  if (!c || !d_queries || !key_slots || !d_rows || !B || !d0 || !d1 || (d1 & (d1 - 1)))
    FAIL(GPIR_INVALID_ARGUMENT, "invalid sharded expansion input");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  cudaStream_t s = pick_stream(c, stream);
  int rc;
  switch (c->logn * 10000 + c->k * 100 + c->ell) {
    GPIR_COMBOS(DISPATCH_CASE_SHX)
    default:
      FAIL(GPIR_UNSUPPORTED, "unsupported combination");
  }
  if (rc) return rc;
  if (!stream) CK(cudaStreamSynchronize(s));
  return 0;
}

int gpir_sharded_rowsel(gpir_ctx* c, const gpir_db* db, const uint32_t* d_rows, uint32_t B, uint32_t* d_partial,
                        void* stream) {
  if (!c || !db || !d_rows || !d_partial || !B) FAIL(GPIR_INVALID_ARGUMENT, "invalid sharded rowsel input");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  cudaStream_t s = pick_stream(c, stream);
  int rc;
  uint32_t launches = 0;
  gpir_db* mdb = const_cast<gpir_db*>(db);
  switch (c->logn * 10000 + c->k * 100 + c->ell) {
    case 120405: rc = Engine<12, 4, 5>::rowsel(c, d_rows, (size_t)db->d0 * c->ct_words(), (int)B, mdb, d_partial, s, &launches); break;
    case 80205: rc = Engine<8, 2, 5>::rowsel(c, d_rows, (size_t)db->d0 * c->ct_words(), (int)B, mdb, d_partial, s, &launches); break;
    case 60206: rc = Engine<6, 2, 6>::rowsel(c, d_rows, (size_t)db->d0 * c->ct_words(), (int)B, mdb, d_partial, s, &launches); break;
    default: FAIL(GPIR_UNSUPPORTED, "unsupported combination");
  }
  if (rc) return rc;
  if (!stream) CK(cudaStreamSynchronize(s));
  return 0;
}

#define DISPATCH_CASE_SHR(L, K_, E) \
  case L * 10000 + K_ * 100 + E:    \
    rc = Engine<L, K_, E>::sh_rgsw(c, bit_lo, bit_hi, d_rgsw, s); break;

int gpir_sharded_rgsw(gpir_ctx* c, uint32_t bit_lo, uint32_t bit_hi, uint32_t* d_rgsw, void* stream) {
  if (!c || !d_rgsw) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  cudaStream_t s = pick_stream(c, stream);
  int rc;
  switch (c->logn * 10000 + c->k * 100 + c->ell) {
    GPIR_COMBOS(DISPATCH_CASE_SHR)
    default:
      FAIL(GPIR_UNSUPPORTED, "unsupported combination");
  }
  if (rc) return rc;
  if (!stream) CK(cudaStreamSynchronize(s));
  return 0;
}

int gpir_layout_convert(gpir_ctx* c, const uint32_t* d_in, uint32_t* d_out, uint64_t polys, void* stream) {
  if (!c || !d_in || !d_out) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  cudaStream_t s = pick_stream(c, stream);
  int rc = bitrev_rows(c, d_in, d_out, (size_t)polys * c->k, s);
  if (rc) return rc;
  if (!stream) CK(cudaStreamSynchronize(s));
  return 0;
}

#define DISPATCH_CASE_SHC(L, K_, E) \
  case L * 10000 + K_ * 100 + E:    \
    rc = Engine<L, K_, E>::sh_coltor(c, d_sums, (int)B, d_out, s); break;

int gpir_sharded_coltor(gpir_ctx* c, uint32_t* d_sums, uint32_t B, uint32_t* d_out, void* stream) {
  if (!c || !d_sums || !d_out || !B) FAIL(GPIR_INVALID_ARGUMENT, "invalid sharded coltor input");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  cudaStream_t s = pick_stream(c, stream);
  int rc;
  switch (c->logn * 10000 + c->k * 100 + c->ell) {
    GPIR_COMBOS(DISPATCH_CASE_SHC)
    default:
      FAIL(GPIR_UNSUPPORTED, "unsupported combination");
  }
  if (rc) return rc;
  if (!stream) CK(cudaStreamSynchronize(s));
  return 0;
}

#define DISPATCH_CASE_CT(L, K_, E) \
  case L * 10000 + K_ * 100 + E:   \
    rc = Engine<L, K_, E>::coltor_dev(c, d_cts, (int)B, (int)C, d_rgsw, d_out, s); break;

int gpir_sharded_rowsel_coltor(gpir_ctx* c, const gpir_db* db, const uint32_t* d_rows, uint32_t B,
                               const uint32_t* d_rgsw_low, uint32_t* d_out, void* stream) {
  if (!c || !db || !d_rows || !d_out || !B) FAIL(GPIR_INVALID_ARGUMENT, "invalid sharded rowsel/coltor input");
  if (db->d1 > 1 && !d_rgsw_low) FAIL(GPIR_INVALID_ARGUMENT, "missing low-bit RGSW rows");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  cudaStream_t s = pick_stream(c, stream);
  int rc;
  gpir_db* mdb = const_cast<gpir_db*>(db);
  switch (c->logn * 10000 + c->k * 100 + c->ell) {
    case 120405: rc = Engine<12, 4, 5>::rowsel_coltor(c, mdb, d_rows, (int)B, d_rgsw_low, d_out, s); break;
    case 80205: rc = Engine<8, 2, 5>::rowsel_coltor(c, mdb, d_rows, (int)B, d_rgsw_low, d_out, s); break;
    case 60206: rc = Engine<6, 2, 6>::rowsel_coltor(c, mdb, d_rows, (int)B, d_rgsw_low, d_out, s); break;
    default: FAIL(GPIR_UNSUPPORTED, "unsupported combination");
  }
  if (rc) return rc;
  if (!stream) CK(cudaStreamSynchronize(s));
  return 0;
}

int gpir_coltor_dev(gpir_ctx* c, const uint32_t* d_cts, uint32_t B, uint32_t C, const uint32_t* d_rgsw,
                    uint32_t* d_out, void* stream) {
  if (!c || !d_cts || !d_out || !C || (C & (C - 1))) FAIL(GPIR_INVALID_ARGUMENT, "invalid tournament input");
  std::lock_guard<std::mutex> lk(c->mu);
  cudaGetLastError();  // a stale non-sticky error of an earlier call must not fail this one
  CK(cudaSetDevice(c->device));
  cudaStream_t s = pick_stream(c, stream);
  int rc;
  switch (c->logn * 10000 + c->k * 100 + c->ell) {
    GPIR_COMBOS(DISPATCH_CASE_CT)
    default:
      FAIL(GPIR_UNSUPPORTED, "unsupported combination");
  }
  if (rc) return rc;
  if (!stream) CK(cudaStreamSynchronize(s));
  return 0;
}

#define OP_DISPATCH(CALL)                                                   \
  std::lock_guard<std::mutex> lk(c->mu);                                    \
  cudaGetLastError();                                                       \
  CK(cudaSetDevice(c->device));                                             \
  switch (c->logn * 10000 + c->k * 100 + c->ell) {                          \
    case 120405: return Engine<12, 4, 5>::CALL;                             \
    case 80205: return Engine<8, 2, 5>::CALL;                               \
    case 60206: return Engine<6, 2, 6>::CALL;                               \
    default: FAIL(GPIR_UNSUPPORTED, "unsupported combination");             \
  }

int gpir_op_ntt(gpir_ctx* c, const uint32_t* in, uint32_t* out, uint32_t polys, int inverse) {
  if (!c || !in || !out) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  if (!polys) return 0;
  OP_DISPATCH(op_ntt(c, in, out, polys, inverse));
}

int gpir_op_digits(gpir_ctx* c, const uint32_t* coeff, int32_t* digits_out, uint32_t polys) {
  if (!c || !coeff || !digits_out) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  if (!polys) return 0;
  OP_DISPATCH(op_digits(c, coeff, digits_out, polys));
}

int gpir_op_expand_stage(gpir_ctx* c, const uint32_t* state, uint32_t B, uint32_t C, const uint32_t* ksk,
                         uint32_t stage, int mode, uint32_t* out) {
  if (!c || !state || !ksk || !out || !B || !C) FAIL(GPIR_INVALID_ARGUMENT, "invalid expand_stage input");
  if (stage >= c->logn) FAIL(GPIR_INVALID_ARGUMENT, "stage out of range");
  OP_DISPATCH(op_expand_stage(c, state, (int)B, (int)C, ksk, (int)stage, mode, out));
}

int gpir_op_ext_product(gpir_ctx* c, const uint32_t* cts, uint32_t B, uint32_t M, const uint32_t* rows, int mode,
                        uint32_t* out) {
  if (!c || !cts || !rows || !out) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  if (!B || !M) return 0;
  OP_DISPATCH(op_xp(c, cts, (int)B, (int)M, 0, rows, mode, out));
}

int gpir_op_coltor_stage(gpir_ctx* c, const uint32_t* state, uint32_t B, uint32_t C, const uint32_t* rows, int mode,
                         uint32_t* out) {
  if (!c || !state || !rows || !out || C < 2 || (C & 1)) FAIL(GPIR_INVALID_ARGUMENT, "invalid tournament stage input");
  OP_DISPATCH(op_xp(c, state, (int)B, (int)(C / 2), 1, rows, mode, out));
}

int gpir_op_rowsel(gpir_ctx* c, const uint32_t* row_cts, uint32_t B, const gpir_db* db, uint32_t* selected) {
  if (!c || !row_cts || !db || !selected) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  if (!B) return 0;
  OP_DISPATCH(op_rowsel(c, row_cts, (int)B, const_cast<gpir_db*>(db), selected));
}

}  // extern "C"
