/*
 * gpir.h — C ABI of the B200-native GPIR server pipeline (libgpir.so).
 *
 * Drop-in boundary for the reference's server path (`latpir`, Python):
 *   encode_database  src/protocol.py:118-153   -> gpir_db_encode / gpir_db_upload
 *   ClientKeys upload (evk_raw / sk_rgsw_raw)
 *                    src/protocol.py:165-199   -> gpir_keys_put
 *   answer_batch     src/protocol.py:635-682   -> gpir_answer_batch (host buffers)
 *                                               gpir_answer_batch_dev (device buffers)
 *   cluster._answer_shard src/cluster.py:252-265 -> gpir_shard_answer
 *   col_tournament_batch src/protocol.py:542-573 -> gpir_coltor_dev
 *   wire.deserialize_query / serialize_response / deserialize_evkset
 *                    src/wire.py:263-318   -> gpir_wire_* (batch collector codec)
 *   wire.save_database / load_database
 *                    src/wire.py:365-410   -> gpir_db_save / gpir_db_load
 * Operator-level parity entry points (host buffers, reference natural order):
 *   ntt_raw / intt_raw      src/ring.py:408-453     -> gpir_op_ntt
 *   DigitExtractor          src/he.py:323-367       -> gpir_op_digits
 *   planner.expand_stage    src/planner.py:321-381  -> gpir_op_expand_stage
 *   planner.external_product_batch src/planner.py:384-435 -> gpir_op_ext_product
 *   planner.coltor_stage    src/planner.py:438-463  -> gpir_op_coltor_stage
 *   layout.gemm_* (p-major) src/layout.py:190-294   -> gpir_op_rowsel
 *
 * Conventions: all residues are uint32 canonical (< q_i < 2^31); every
 * ciphertext is [2][k][n] (a then b), every polynomial [k][n], NTT-domain
 * values in the reference's NATURAL slot order at this boundary.  Functions
 * return 0 on success, a negative gpir_status otherwise; gpir_last_error()
 * gives the message (thread-local).  Contexts are thread-safe (one internal
 * mutex per context).  Stage modes: 0 = operation-level, 1 = stage-fused
 * (planner.ExecMode OPERATION_LEVEL / STAGE_LEVEL, src/planner.py:105-107),
 * 2 = split stage-fused (per-node iNTT+Dcp kernel, per node x limb NTT+MAC
 * kernel), 3 = hybrid (operation-level iNTT and Dcp, then the per node x limb
 * NTT+MAC kernel); all bit-identical.  Key rows are stored with the top gadget
 * digit folded in (see k_fold_rows), so ell-1 digits per component are
 * transformed.
 */
#ifndef GPIR_H
#define GPIR_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gpir_ctx gpir_ctx;
typedef struct gpir_db gpir_db;

enum gpir_status {
  GPIR_OK = 0,
  GPIR_INVALID_ARGUMENT = -1, /* latpir.errors.InvalidArgument */
  GPIR_INVALID_STATE = -2,    /* latpir.errors.InvalidState    */
  GPIR_INVALID_CONFIG = -3,   /* latpir.errors.InvalidConfig   */
  GPIR_CUDA_ERROR = -4,
  GPIR_UNSUPPORTED = -5,
  GPIR_PARSE_ERROR = -6       /* latpir.errors.ParseError; offset: gpir_last_error_offset() */
};

typedef struct gpir_stats {
  float ms_expand;   /* ExpandQuery                     */
  float ms_rgsw;     /* RGSW assembly                   */
  float ms_rowsel;   /* RowSel                          */
  float ms_coltor;   /* ColTor                          */
  float ms_total;    /* device time of the whole batch  */
  float ms_h2d;      /* host->device of queries (host API only) */
  float ms_d2h;      /* device->host of responses (host API only) */
  uint32_t launches; /* kernels launched for the batch  */
  float ms_rowsel_kernel; /* RowSel GEMM kernel alone      */
  float ms_rowsel_transpose; /* RowSel output transpose (P-major -> ciphertexts), 0 if none */
} gpir_stats;

/* Per-stage device time of the last batch (gpir_set_stage_timing on): one
 * entry per ExpandQuery stage, RGSW assembly, RowSel (incl. the operand pack)
 * and ColTor stage, from CUDA events on the launch stream. */
typedef struct gpir_stage_time {
  uint8_t phase;  /* 0 ExpandQuery, 1 RgswAssembly, 2 RowSel, 3 ColTor */
  uint8_t mode;   /* executor mode of the stage (see header comment) */
  uint16_t stage; /* stage index within the phase */
  uint32_t units; /* nodes / ciphertexts / queries processed by the stage (whole batch) */
  float ms;
} gpir_stage_time;

const char* gpir_last_error(void);
/* byte offset of the last GPIR_PARSE_ERROR (ParseError.offset) */
int64_t gpir_last_error_offset(void);
const char* gpir_version(void);

/* Context: ring degree n (power of two), k primes q[i] with 2n-th roots psi[i]
 * (src/ring.py:122-158), gadget z = 2^z_bits with ell digits (src/he.py:45-55). */
gpir_ctx* gpir_ctx_create(int device, uint32_t n, uint32_t k, const uint32_t* q, const uint32_t* psi,
                          uint32_t z_bits, uint32_t ell);
void gpir_ctx_destroy(gpir_ctx* ctx);
int gpir_ctx_device(const gpir_ctx* ctx);
/* RowSel engine: 0 = auto (tensor cores when d0 <= 1024; A tiles of 128 rows),
 * 1 = CUDA cores (64-bit lazy IMAD), 2 = tensor cores (tcgen05 kind::i8). */
int gpir_set_rowsel_engine(gpir_ctx* ctx, int engine);

/* CUDA-graph replay of the device pipeline (default on; GPIR_GRAPH=0 in the
 * environment turns it off for new contexts).  Calls without stats and without
 * stage timing record the pipeline of a (db, B, buffers, plan) shape on its
 * second call and replay the graph from the third; any device (re)allocation
 * invalidates the recorded graphs. */
int gpir_set_graphs(gpir_ctx* ctx, int on);
/* Kernels this library has launched eagerly so far, process-wide (launches inside
 * replayed CUDA graphs are not counted). */
uint64_t gpir_launch_count(void);
/* Capacity path knobs (0 = automatic): the bytes the (B, d1) RowSel selection
 * may occupy before RowSel and the low ColTor stages run per power-of-two
 * column window (default 16 GiB), and the largest sub-batch served at once
 * (default: what the free device memory holds).  Results do not change. */
int gpir_set_capacity(gpir_ctx* ctx, uint64_t sel_budget_bytes, uint32_t max_batch);
/* Supported (log2 n, k, ell) combinations are compiled in; 1 if supported. */
int gpir_supported(uint32_t n, uint32_t k, uint32_t ell);

/* Database: d0 x d1 grid of records, row-major flat index r = i*d1 + j
 * (src/protocol.py:58-61).  encode: raw bytes, record_bytes each, packed as
 * little-endian plain_bits/8-byte words, centered mod P, lifted and NTT'd on
 * the GPU (src/protocol.py:102-153).  upload: an already-encoded P-major
 * (d1, d0, k*n) tensor in natural order (EncodedDatabase.data). */
gpir_db* gpir_db_encode(gpir_ctx* ctx, const uint8_t* records, uint32_t d0, uint32_t d1, uint32_t record_bytes,
                        uint32_t plain_bits);
gpir_db* gpir_db_upload(gpir_ctx* ctx, const uint32_t* pmajor, uint32_t d0, uint32_t d1);
/* encode from records already in device memory (d_records: d0*d1*record_bytes
 * bytes on the context's device), e.g. generated on the GPU for DBs of many GiB;
 * same encoding as gpir_db_encode. */
gpir_db* gpir_db_encode_dev(gpir_ctx* ctx, const uint8_t* d_records, uint32_t d0, uint32_t d1, uint32_t record_bytes,
                            uint32_t plain_bits);
/* Capacity mode: keep only the tensor-core byte-plane image of the DB (the
 * TMEM-resident RowSel layout) and release the u32 copy, so the DB occupies its
 * encoded size once in HBM (configs 4-5).  Needs d0 <= 256.  A compact DB
 * cannot be downloaded or saved (GPIR_INVALID_STATE). */
int gpir_db_compact(gpir_ctx* ctx, gpir_db* db);
/* GPDB container (wire.save_database / load_database, src/wire.py:365-410):
 * load validates magic, version and the primes against the context (and the
 * plain modulus when expect_plain_bits != 0), streams the payload to the GPU
 * and transposes a TRANSPOSED image there; errors are GPIR_PARSE_ERROR with the
 * reference's message and offset.  save writes a P-major image. */
gpir_db* gpir_db_load(gpir_ctx* ctx, const char* path, uint32_t expect_plain_bits, uint32_t* d0, uint32_t* d1,
                      uint32_t* record_bytes, uint32_t* plain_bits);
int gpir_db_save(gpir_ctx* ctx, const gpir_db* db, const char* path, uint32_t record_bytes, uint32_t plain_bits);
/* Download the encoded DB back as the reference's P-major natural tensor. */
int gpir_db_download(gpir_ctx* ctx, const gpir_db* db, uint32_t* pmajor_out);
void gpir_db_destroy(gpir_ctx* ctx, gpir_db* db);
size_t gpir_db_bytes(const gpir_db* db); /* device bytes held (u32 image + byte planes) */

/* Client key material, stored in key slot `slot`: evks[stages][ell][2][k][n]
 * (stage t uses k_aut = n/2^t + 1, src/he.py:225-241) and sk_rgsw[2 ell][2][k][n]
 * (may be NULL when the DB has one column). */
int gpir_keys_put(gpir_ctx* ctx, int slot, const uint32_t* evks, uint32_t stages, const uint32_t* sk_rgsw);
int gpir_keys_drop(gpir_ctx* ctx, int slot);

/* ---- client-side material on the GPU (benchmark input factory; src/he.py:220-271,
 * 423-431, 487-515, src/protocol.py:240-281) ----
 * keygen samples a ternary secret and encrypts the `stages` expansion keys and
 * RGSW(s) with errors of the given bound (a counter-based RNG keyed by seed, so
 * samples differ from numpy's, distributions and equations do not), installs
 * them in key slot `slot`, and returns the secret's coefficients (int8, n) for
 * client-side decryption.  queries encrypts (i*, j*) pairs under that secret:
 * queries_out[count][2][k][n] host, natural order. */
int gpir_client_keygen(gpir_ctx* ctx, int slot, uint32_t stages, uint64_t seed, uint32_t error_bound,
                       int8_t* secret_out);
int gpir_client_queries(gpir_ctx* ctx, const int8_t* secret, uint32_t plain_bits, uint32_t error_bound, uint32_t d0,
                        uint32_t d1, const uint32_t* i_star, const uint32_t* j_star, uint32_t count, uint64_t seed,
                        uint32_t* queries_out);

/* Full server pipeline for B queries (src/protocol.py:635-682).
 * queries[B][2][k][n] host; key_slots[B]; modes: one byte per ExpandQuery stage
 * (n_eq) and per ColTor stage (n_ct), or NULL for the built-in B200 plan;
 * responses_out[B][2][k][n] host.  stats may be NULL. */
int gpir_answer_batch(gpir_ctx* ctx, const gpir_db* db, const uint32_t* queries, const int32_t* key_slots,
                      uint32_t B, const uint8_t* eq_modes, uint32_t n_eq, const uint8_t* ct_modes, uint32_t n_ct,
                      uint32_t* responses_out, gpir_stats* stats);
/* Same with device pointers (natural order in/out) on `stream` (cudaStream_t or NULL). */
int gpir_answer_batch_dev(gpir_ctx* ctx, const gpir_db* db, const uint32_t* d_queries, const int32_t* key_slots,
                          uint32_t B, const uint8_t* eq_modes, uint32_t n_eq, const uint8_t* ct_modes, uint32_t n_ct,
                          uint32_t* d_responses, void* stream, gpir_stats* stats);

int gpir_set_stage_timing(gpir_ctx* ctx, int on);
/* copies up to cap entries of the last timed batch; returns the entry count (>= 0) */
int gpir_stage_times(gpir_ctx* ctx, gpir_stage_time* out, uint32_t cap);

/* Built-in B200 hybrid plan (per-stage op/fused choice) for a geometry/batch. */
int gpir_plan(gpir_ctx* ctx, uint32_t d0, uint32_t d1, uint32_t B, uint8_t* eq_modes, uint32_t n_eq,
              uint8_t* ct_modes, uint32_t n_ct);

/* ---- sharded pipeline pieces (multi-GPU, D1 column shards; src/cluster.py:252-265) ----
 * gpir_shard_answer: expansion over the FULL geometry (d0, d1_total), RowSel +
 * the low log2(d1_shard) ColTor stages on the local column shard (db holds
 * d1_shard columns), writes one partial ct per query (natural order) to
 * d_partials[B][2][k][n] and the high-bit RGSWs (natural order) to
 * d_high_rgsw[B][log2(d1_total/d1_shard)][2 ell][2][k][n] (may be NULL). */
int gpir_shard_answer(gpir_ctx* ctx, const gpir_db* db, uint32_t d1_total, const uint32_t* d_queries,
                      const int32_t* key_slots, uint32_t B, uint32_t* d_partials, uint32_t* d_high_rgsw,
                      void* stream, gpir_stats* stats);
/* Column-sharded worker step (the reference's _Worker._answer_shard,
 * src/cluster.py:252-265): RowSel of B queries' row cts d_rows (internal
 * layout, (B, d0) from gpir_sharded_expand) against this shard's columns and
 * the shard's log2(d1) low ColTor stages with d_rgsw_low (B, log2 d1, 2 ell,
 * 2, k, n) -> d_out (B, 2, k, n).  Large shards run per column window. */
int gpir_sharded_rowsel_coltor(gpir_ctx* ctx, const gpir_db* db, const uint32_t* d_rows, uint32_t B,
                               const uint32_t* d_rgsw_low, uint32_t* d_out, void* stream);
/* Residual tournament: d_cts[B][C][2][k][n] (C power of two) with
 * d_rgsw[B][log2 C][2 ell][2][k][n], natural order -> d_out[B][2][k][n]. */
int gpir_coltor_dev(gpir_ctx* ctx, const uint32_t* d_cts, uint32_t B, uint32_t C, const uint32_t* d_rgsw,
                    uint32_t* d_out, void* stream);

/* ---- row-sharded pipeline (D0 shards + modular-add combine; north-star
 * multi-GPU mode).  Per rank r of n (device buffers, `stream` or NULL):
 *   1. gpir_sharded_expand: expand the rank's OWN queries (B_own) over the full
 *      (d0, d1) tree and assemble their RGSWs; writes their row ciphertexts
 *      d_rows[B_own][d0][2][k][n] (internal brv slot order).  The expansion and
 *      RGSWs stay in the context for step 3.
 *   2. (caller) all-to-all of row blocks so every rank holds all B queries'
 *      rows of its own D0 range; gpir_sharded_rowsel multiplies them with the
 *      local DB rows (db has d0/n rows x d1 columns) -> d_partial[B][d1][2][k][n].
 *   3. (caller) reduce-scatter(sum, int32) of the partials by query owner;
 *      gpir_sharded_coltor reduces the sums mod q in place and runs the
 *      tournament for the own queries -> d_out[B_own][2][k][n] (natural order). */
int gpir_sharded_expand(gpir_ctx* ctx, uint32_t d0, uint32_t d1, const uint32_t* d_queries, const int32_t* key_slots,
                        uint32_t B_own, uint32_t* d_rows, void* stream);
int gpir_sharded_rowsel(gpir_ctx* ctx, const gpir_db* db, const uint32_t* d_rows, uint32_t B, uint32_t* d_partial,
                        void* stream);
int gpir_sharded_coltor(gpir_ctx* ctx, uint32_t* d_sums, uint32_t B_own, uint32_t* d_out, void* stream);
/* Column-sharded mode (src/cluster.py SHARD_ALL_GATHER over NCCL): after
 * gpir_sharded_expand, export the own queries' RGSW rows of column bits
 * [bit_lo, bit_hi) in natural order as d_rgsw[B_own][bit_hi-bit_lo][2 ell][2][k][n]
 * (the layout gpir_coltor_dev takes). */
int gpir_sharded_rgsw(gpir_ctx* ctx, uint32_t bit_lo, uint32_t bit_hi, uint32_t* d_rgsw, void* stream);
/* natural <-> internal bit-reversed slot order of `polys` ciphertext halves
 * ([polys][k][n] words; an involution), device buffers. */
int gpir_layout_convert(gpir_ctx* ctx, const uint32_t* d_in, uint32_t* d_out, uint64_t polys, void* stream);

/* ---- wire codec (src/wire.py; host only, usable without a GPU) ----
 * A batch collector decodes the framed query messages of a batch straight into
 * one contiguous host buffer queries[count][2][k][n] (pass it pinned to
 * gpir_answer_batch) and encodes responses back into framed bytes, with the
 * reference's validation and ParseError offsets.  bad_index (may be NULL)
 * receives the index of the message being decoded when an error occurs. */
int gpir_wire_parse_header(const uint8_t* buf, size_t len, uint32_t* kind, uint64_t* payload_len);
int gpir_wire_decode_queries(const uint8_t* const* msgs, const size_t* lens, uint32_t count, uint32_t n, uint32_t k,
                             uint32_t* queries, uint64_t* client_ids, uint32_t* seqs, uint32_t* bad_index);
size_t gpir_wire_response_bytes(uint32_t n, uint32_t k);
int gpir_wire_encode_responses(const uint32_t* responses, const uint64_t* client_ids, const uint32_t* seqs,
                               uint32_t count, uint32_t n, uint32_t k, uint8_t* out, size_t out_cap);
/* KIND_EVKSET (serialize_evkset) -> gpir_keys_put layout: evks[stages][ell][2][k][n]
 * by stage (k_aut = n/2^t + 1), sk_rgsw[2 ell][2][k][n] (may be NULL). */
int gpir_wire_decode_evkset(const uint8_t* msg, size_t len, uint32_t n, uint32_t k, uint32_t z_bits, uint32_t ell,
                            uint32_t stages, uint32_t* evks, uint32_t* sk_rgsw, uint64_t* client_id, int* has_rgsw);

/* ---- operator-level parity entry points (host buffers, natural order) ---- */
int gpir_op_ntt(gpir_ctx* ctx, const uint32_t* in, uint32_t* out, uint32_t polys, int inverse);
int gpir_op_digits(gpir_ctx* ctx, const uint32_t* coeff, int32_t* digits_out, uint32_t polys);
int gpir_op_expand_stage(gpir_ctx* ctx, const uint32_t* state, uint32_t B, uint32_t C, const uint32_t* ksk,
                         uint32_t stage, int mode, uint32_t* out /* [B][2C] */);
int gpir_op_ext_product(gpir_ctx* ctx, const uint32_t* cts, uint32_t B, uint32_t M, const uint32_t* rows,
                        int mode, uint32_t* out);
int gpir_op_coltor_stage(gpir_ctx* ctx, const uint32_t* state, uint32_t B, uint32_t C, const uint32_t* rows,
                         int mode, uint32_t* out /* [B][C/2] */);
int gpir_op_rowsel(gpir_ctx* ctx, const uint32_t* row_cts /* [B][d0][2][k][n] */, uint32_t B, const gpir_db* db,
                   uint32_t* selected /* [B][d1][2][k][n] */);

#ifdef __cplusplus
}
#endif
#endif /* GPIR_H */
