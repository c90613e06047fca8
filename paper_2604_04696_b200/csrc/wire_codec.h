// Host-side wire codec for the server path (src/wire.py), compiled into
// libgpir.so (included by gpir.cu, shares its thread-local error state).
//
// The reference decodes every query message into Python objects (header,
// geometry echo, per-limb numpy arrays) and restacks them into the batch
// tensor; a batch collector here decodes the framed bytes of a whole batch
// straight into one contiguous (pinned) host buffer in the layout
// gpir_answer_batch consumes, and encodes the responses back into framed
// bytes without intermediate objects.  Validation and error offsets follow
// the reference exactly (src/wire.py:59-80, 83-100, 145-158, 263-279), so a
// malformed message raises the same ParseError at the same offset.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

namespace gpir_wire {

constexpr char kMagic[4] = {'G', 'P', 'I', 'R'};
constexpr char kDbMagic[4] = {'G', 'P', 'D', 'B'};
constexpr uint16_t kVersion = 1;
constexpr size_t kHeader = 15;  // magic[4] version u16 kind u8 length u64
constexpr size_t kEcho = 6;     // n u32, k u8, domain u8
constexpr size_t kRoute = 12;   // client_id u64, seq u32
enum Kind : uint32_t { kParams = 1, kQuery = 2, kEvkset = 3, kResponse = 4, kError = 5, kCt = 17 };

static thread_local int64_t g_off = 0;

inline int parse_fail(const std::string& msg, int64_t off);

template <class T>
inline T rd(const uint8_t* p) {
  T v;
  memcpy(&v, p, sizeof(T));  // little-endian host (x86-64 / aarch64)
  return v;
}
template <class T>
inline void wr(uint8_t* p, T v) {
  memcpy(p, &v, sizeof(T));
}

// parse_header (src/wire.py:59-69)
inline int header(const uint8_t* buf, size_t len, uint32_t* kind, uint64_t* plen) {
  if (len < kHeader) return parse_fail("truncated header", (int64_t)len);
  if (memcmp(buf, kMagic, 4) != 0) {
    char m[64];
    snprintf(m, sizeof m, "bad magic b'%c%c%c%c'", buf[0], buf[1], buf[2], buf[3]);
    return parse_fail(m, 0);
  }
  const uint16_t ver = rd<uint16_t>(buf + 4);
  if (ver != kVersion) return parse_fail("unsupported version " + std::to_string(ver), 4);
  *kind = buf[6];
  *plen = rd<uint64_t>(buf + 7);
  return 0;
}

// split_message (src/wire.py:72-80) + kind check
inline int payload(const uint8_t* buf, size_t len, uint32_t want, const char* what, const uint8_t** pl,
                   size_t* plen) {
  uint32_t kind;
  uint64_t L;
  int rc = header(buf, len, &kind, &L);
  if (rc) return rc;
  if (len != kHeader + L)
    return parse_fail("payload length mismatch: header says " + std::to_string(L) + ", got " +
                          std::to_string(len - kHeader),
                      (int64_t)kHeader);
  if (kind != want) return parse_fail(std::string("expected ") + what + " message, got kind " + std::to_string(kind), 6);
  *pl = buf + kHeader;
  *plen = (size_t)L;
  return 0;
}

// _read_ct (src/wire.py:145-158) at payload offset off: 2 x k x n words -> out
inline int read_ct(const uint8_t* pl, size_t plen, size_t& off, uint32_t n, uint32_t k, uint32_t* out) {
  if (off + kEcho > plen) return parse_fail("truncated payload", (int64_t)off);
  const uint32_t en = rd<uint32_t>(pl + off);
  const uint32_t ek = pl[off + 4];
  off += kEcho;
  if (en != n || ek != k)
    return parse_fail("geometry echo (" + std::to_string(en) + ", " + std::to_string(ek) +
                          ") does not match basis (" + std::to_string(n) + ", " + std::to_string(k) + ")",
                      (int64_t)(off - kEcho));
  const size_t bytes = (size_t)2 * k * n * 4;
  if (off + bytes > plen) {
    // the reference takes the two components one at a time
    const size_t one = (size_t)k * n * 4;
    return parse_fail("truncated payload", (int64_t)(off + (off + one <= plen ? one : 0)));
  }
  memcpy(out, pl + off, bytes);
  off += bytes;
  return 0;
}

}  // namespace gpir_wire

extern "C" {

int64_t gpir_last_error_offset(void) { return gpir_wire::g_off; }

size_t gpir_wire_response_bytes(uint32_t n, uint32_t k) {
  return gpir_wire::kHeader + gpir_wire::kRoute + gpir_wire::kEcho + (size_t)2 * k * n * 4;
}

int gpir_wire_parse_header(const uint8_t* buf, size_t len, uint32_t* kind, uint64_t* payload_len) {
  if (!buf || !kind || !payload_len) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  return gpir_wire::header(buf, len, kind, payload_len);
}

int gpir_wire_decode_queries(const uint8_t* const* msgs, const size_t* lens, uint32_t count, uint32_t n, uint32_t k,
                             uint32_t* cts, uint64_t* client_ids, uint32_t* seqs, uint32_t* bad_index) {
  using namespace gpir_wire;
  if (!msgs || !lens || (count && (!cts || !client_ids || !seqs))) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  const size_t ct_words = (size_t)2 * k * n;
  for (uint32_t i = 0; i < count; ++i) {
    if (bad_index) *bad_index = i;
    const uint8_t* pl;
    size_t plen;
    int rc = payload(msgs[i], lens[i], kQuery, "query", &pl, &plen);
    if (rc) return rc;
    if (plen < kRoute) return parse_fail("truncated payload", 0);
    client_ids[i] = rd<uint64_t>(pl);
    seqs[i] = rd<uint32_t>(pl + 8);
    size_t off = kRoute;
    if ((rc = read_ct(pl, plen, off, n, k, cts + (size_t)i * ct_words))) return rc;
    if (off != plen) return parse_fail("trailing bytes after value", (int64_t)off);
  }
  return 0;
}

int gpir_wire_encode_responses(const uint32_t* cts, const uint64_t* client_ids, const uint32_t* seqs, uint32_t count,
                               uint32_t n, uint32_t k, uint8_t* out, size_t out_cap) {
  using namespace gpir_wire;
  const size_t each = gpir_wire_response_bytes(n, k);
  if ((count && (!cts || !client_ids || !seqs || !out)) || out_cap < each * count)
    FAIL(GPIR_INVALID_ARGUMENT, "response buffer too small");
  const size_t ct_words = (size_t)2 * k * n;
  for (uint32_t i = 0; i < count; ++i) {  // serialize_response (src/wire.py:282-283)
    uint8_t* m = out + each * i;
    memcpy(m, kMagic, 4);
    wr<uint16_t>(m + 4, kVersion);
    m[6] = (uint8_t)kResponse;
    wr<uint64_t>(m + 7, (uint64_t)(each - kHeader));
    wr<uint64_t>(m + 15, client_ids[i]);
    wr<uint32_t>(m + 23, seqs[i]);
    wr<uint32_t>(m + 27, n);
    m[31] = (uint8_t)k;
    m[32] = 1;  // NTT domain
    memcpy(m + 33, cts + (size_t)i * ct_words, ct_words * 4);
  }
  return 0;
}

// Evaluation-key set (serialize_evkset, src/wire.py:296-318) decoded into the
// gpir_keys_put layout: evks[stages][ell][2][k][n] ordered by stage t (k_aut =
// n/2^t + 1) and sk_rgsw[2 ell][2][k][n].  `stages` is how many the caller
// wants; every stage must be present in the message.
int gpir_wire_decode_evkset(const uint8_t* msg, size_t len, uint32_t n, uint32_t k, uint32_t z_bits, uint32_t ell,
                            uint32_t stages, uint32_t* evks, uint32_t* sk_rgsw, uint64_t* client_id,
                            int* has_rgsw) {
  using namespace gpir_wire;
  if (!msg || !client_id || !has_rgsw || (stages && !evks)) FAIL(GPIR_INVALID_ARGUMENT, "null argument");
  const uint8_t* pl;
  size_t plen;
  int rc = payload(msg, len, kEvkset, "evkset", &pl, &plen);
  if (rc) return rc;
  if (plen < 11) return parse_fail("truncated payload", 0);
  *client_id = rd<uint64_t>(pl);
  const uint32_t count = rd<uint16_t>(pl + 8);
  *has_rgsw = pl[10] ? 1 : 0;
  size_t off = 11;
  const size_t ctw = (size_t)2 * k * n;
  uint64_t seen = 0;
  for (uint32_t e = 0; e < count; ++e) {
    if (off + 7 > plen) return parse_fail("truncated payload", (int64_t)off);
    const uint32_t k_aut = rd<uint32_t>(pl + off);
    const uint32_t zb = pl[off + 4], el = rd<uint16_t>(pl + off + 5);
    off += 7;
    if (zb != z_bits || el != ell)
      return parse_fail("evaluation key gadget does not match the server profile", (int64_t)(off - 7));
    int t = -1;
    for (uint32_t s = 0; s < stages && s < 64; ++s)
      if (k_aut == n / (1u << s) + 1) t = (int)s;
    for (uint32_t r = 0; r < el; ++r) {
      uint32_t* dst = t >= 0 ? evks + ((size_t)t * ell + r) * ctw : nullptr;
      if (dst) {
        if ((rc = read_ct(pl, plen, off, n, k, dst))) return rc;
      } else {  // a key this geometry does not use: validate and skip
        if (off + kEcho > plen) return parse_fail("truncated payload", (int64_t)off);
        if (rd<uint32_t>(pl + off) != n || pl[off + 4] != k)
          return parse_fail("geometry echo does not match basis", (int64_t)off);
        off += kEcho + ctw * 4;
        if (off > plen) return parse_fail("truncated payload", (int64_t)plen);
      }
    }
    if (t >= 0) seen |= 1ull << t;
  }
  for (uint32_t s = 0; s < stages; ++s)
    if (!(seen >> s & 1)) {
      g_err = "evkset lacks the evaluation key for k_aut " + std::to_string(n / (1u << s) + 1);
      return GPIR_INVALID_STATE;
    }
  if (*has_rgsw) {
    if (off + 3 > plen) return parse_fail("truncated payload", (int64_t)off);
    const uint32_t zb = pl[off], el = rd<uint16_t>(pl + off + 1);
    off += 3;
    if (zb != z_bits || el != ell) return parse_fail("RGSW gadget does not match the server profile", (int64_t)(off - 3));
    for (uint32_t r = 0; r < 2 * el; ++r) {
      if (sk_rgsw) {
        if ((rc = read_ct(pl, plen, off, n, k, sk_rgsw + (size_t)r * ctw))) return rc;
      } else {
        off += kEcho + ctw * 4;
        if (off > plen) return parse_fail("truncated payload", (int64_t)plen);
      }
    }
  }
  if (off != plen) return parse_fail("trailing bytes after value", (int64_t)off);
  return 0;
}

}  // extern "C"

namespace gpir_wire {
inline int parse_fail(const std::string& msg, int64_t off) {
  g_err = msg;
  g_off = off;
  return -6;  // GPIR_PARSE_ERROR
}
}  // namespace gpir_wire
