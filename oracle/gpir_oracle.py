"""CPU ORACLE for the GPIR server pipeline — TEST INFRASTRUCTURE ONLY.

This module is a restatement of the reference `latpir` algorithms (arXiv
2604.04696, CPU reference package under /root/reference/pkg/src/latpir) in
numpy (+ numba for the transforms, as the reference itself does).  It exists
to CHECK the CUDA path, and as the `cpu_baseline` / `--impl reference` leg of
bench.py.  Only `tests/`, `__graft_entry__.smoke()` and bench.py's CPU legs may
import it; the product package (`paper_2604_04696_b200`) never does and has no
CPU fallback.

Parity is pinned: `tests/test_oracle.py` checks every function here against
golden vectors produced by running the live reference in the build container
(`tools/make_golden.py` -> `tests/golden/*.npz`).

All arrays are uint64 canonical residues with limb-major (..., k, n) shape, as
in the reference (`src/ring.py:14-16`).  Citations: `src/` =
/root/reference/pkg/src/latpir/.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

U64 = np.uint64

try:  # the reference accelerates its transforms with numba (src/ring.py:37-43)
    if os.environ.get("GPIR_ORACLE_NO_NUMBA"):
        raise ImportError
    import numba as _nb
except ImportError:  # pragma: no cover
    _nb = None


# ---------------------------------------------------------------------------
# primes, roots, basis  (src/ring.py:55-90, 239-263)

def is_prime(v: int) -> bool:
    """Deterministic Miller-Rabin over the first 12 primes (src/ring.py:55-77)."""
    if v < 2:
        return False
    bases = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for p in bases:
        if v % p == 0:
            return v == p
    d, s = v - 1, 0
    while not d & 1:
        d >>= 1
        s += 1
    for a in bases:
        x = pow(a, d, v)
        if x == 1 or x == v - 1:
            continue
        for _ in range(s - 1):
            x = x * x % v
            if x == v - 1:
                break
        else:
            return False
    return True


def two_n_root(q: int, two_n: int) -> int:
    """First g^((q-1)/2n), g = 2, 3, ..., whose n-th power is -1 (src/ring.py:80-90)."""
    cof = (q - 1) // two_n
    for g in range(2, q):
        r = pow(g, cof, q)
        if pow(r, two_n // 2, q) == q - 1:
            return r
    raise ValueError("no root")


class Ring:
    """RNS ring Z_Q[X]/(X^n+1) with transform and CRT tables (src/ring.py:122-235)."""

    def __init__(self, n: int, qs, psis=None):
        self.n = n
        self.logn = n.bit_length() - 1
        self.qs = [int(q) for q in qs]
        self.k = len(self.qs)
        two_n = 2 * n
        self.psis = [int(p) for p in psis] if psis is not None else [two_n_root(q, two_n) for q in self.qs]
        self.Q = math.prod(self.qs)
        self.q = np.array(self.qs, dtype=U64)[:, None]          # (k, 1)
        self.q_i64 = self.q.astype(np.int64)
        # psi^e for e in [0, 2n)
        pw = np.empty((self.k, two_n), dtype=U64)
        for i, (q, psi) in enumerate(zip(self.qs, self.psis)):
            v = 1
            for e in range(two_n):
                pw[i, e] = v
                v = v * psi % q
        self.psi_pow = pw
        # bit reversal permutation
        idx = np.arange(n)
        rev = np.zeros(n, dtype=np.int64)
        for b in range(self.logn):
            rev |= ((idx >> b) & 1) << (self.logn - 1 - b)
        self.bitrev = rev
        # per-stage butterfly twiddles of the natural-order DIT transform:
        # stage with half-size h uses omega^(j * n/(2h)) = psi^(2 j n/(2h))
        self.tw_f, self.tw_i = [], []
        for s in range(self.logn):
            h = 1 << s
            e = (np.arange(h) * (n // h)) % two_n
            self.tw_f.append(pw[:, e][:, None, :])
            self.tw_i.append(pw[:, (two_n - e) % two_n][:, None, :])
        self.twist = np.ascontiguousarray(pw[:, :n])
        untw = np.empty((self.k, n), dtype=U64)
        for i, q in enumerate(self.qs):
            ninv = pow(n, q - 2, q)
            untw[i] = (pw[i, (two_n - np.arange(n)) % two_n].astype(object) * ninv % q).astype(U64)
        self.untwist = untw
        # flat tables for the numba transform (Shoup companions, 32-bit)
        self._flat_f = np.concatenate([t[:, 0, :] for t in self.tw_f], axis=1)
        self._flat_i = np.concatenate([t[:, 0, :] for t in self.tw_i], axis=1)
        sh = lambda tab: np.stack([(tab[i].astype(object) * (1 << 32) // q).astype(U64)
                                   for i, q in enumerate(self.qs)])
        self._flat_f_sh, self._flat_i_sh = sh(self._flat_f), sh(self._flat_i)
        self._twist_sh, self._untwist_sh = sh(self.twist), sh(self.untwist)
        self.jit = _nb is not None and max(self.qs) * (2 * self.logn + 1) < (1 << 32)
        # CRT: y_i = x_i * (Q/q_i)^-1 mod q_i ; X = sum y_i * (Q/q_i)   (src/ring.py:214-235)
        self.crt_m = [self.Q // q for q in self.qs]
        self.crt_mhat = np.array([pow(m % q, q - 2, q) for m, q in zip(self.crt_m, self.qs)], dtype=U64)[:, None]

    @classmethod
    def generate(cls, n: int, k: int, bits: int = 27) -> "Ring":
        """k largest primes q = c*2n+1 below 2^bits, descending (src/ring.py:239-254)."""
        two_n = 2 * n
        qs = []
        c = ((1 << bits) - 2) // two_n
        while len(qs) < k and c > 0:
            q = c * two_n + 1
            if q.bit_length() <= bits and is_prime(q):
                qs.append(q)
            c -= 1
        return cls(n, qs)


@lru_cache(maxsize=None)
def default_ring(n: int = 4096) -> Ring:
    """Production ring: four ~27-bit primes (src/ring.py:260-263)."""
    return Ring.generate(n, 4, 27)


@dataclass
class Params:
    """HeParams restated (src/he.py:45-130): ring, P = 2^plain_bits, gadget (z_bits, ell)."""

    ring: Ring
    plain_bits: int = 32
    z_bits: int = 22
    ell: int = 5
    error_bound: int = 16

    @property
    def n(self):
        return self.ring.n

    @property
    def P(self):
        return 1 << self.plain_bits

    @property
    def delta(self):
        return self.ring.Q // self.P


def default_params(n: int = 4096, plain_bits: int = 32) -> Params:
    """`he.default_params()` (src/he.py:111-114); plain_bits=16 is the D0=256 correctness profile."""
    return Params(default_ring(n), plain_bits)


def test_params(n=256, k=2, prime_bits=27, plain_bits=8, z_bits=11, error_bound=4) -> Params:
    """`he.test_params` (src/he.py:117-130): ell is the least with z^ell > Q."""
    r = Ring.generate(n, k, prime_bits)
    ell = 1
    while (1 << (z_bits * ell)) <= r.Q:
        ell += 1
    return Params(r, plain_bits, z_bits, ell, error_bound)


# ---------------------------------------------------------------------------
# transforms  (src/ring.py:320-453): ntt(a)[j] = a(psi^(2j+1)), natural order

if _nb is not None:

    @_nb.njit(parallel=True, cache=True, nogil=True)
    def _rows_jit(rows, k, rev, tw_pre, tw_pre_sh, tw, tw_sh, qs, inverse):  # pragma: no cover
        n = rows.shape[1]
        out = np.empty_like(rows)
        for r in _nb.prange(rows.shape[0]):
            li = r % k
            q = qs[li]
            buf = np.empty(n, dtype=np.uint64)
            for i in range(n):
                src = rev[i]
                v = rows[r, src]
                if not inverse:
                    t = v * tw_pre[li, src] - ((v * tw_pre_sh[li, src]) >> 32) * q
                    v = t - q if t >= q else t
                buf[i] = v
            base = 0
            h = 1
            while h < n:
                for blk in range(0, n, 2 * h):
                    for j in range(h):
                        w = tw[li, base + j]
                        u = buf[blk + j]
                        x = buf[blk + h + j]
                        t = x * w - ((x * tw_sh[li, base + j]) >> 32) * q
                        buf[blk + j] = u + t
                        buf[blk + h + j] = u + 2 * q - t
                base += h
                h *= 2
            for i in range(n):
                v = buf[i]
                if inverse:
                    t = v * tw_pre[li, i] - ((v * tw_pre_sh[li, i]) >> 32) * q
                    out[r, i] = t - q if t >= q else t
                else:
                    out[r, i] = v % q
        return out


def _ntt_numpy(x, R: Ring, inverse: bool):
    q = R.q
    y = x if inverse else x * R.twist % q
    y = np.ascontiguousarray(y[..., R.bitrev])
    n = R.n
    tws = R.tw_i if inverse else R.tw_f
    for s in range(R.logn):
        h = 1 << s
        v = y.reshape(y.shape[:-1] + (n // (2 * h), 2 * h))
        lo, hi = v[..., :h], v[..., h:]
        qq = q[..., None]
        t = hi * tws[s] % qq
        a = lo + t
        b = lo + qq - t
        v[..., :h] = np.where(a >= qq, a - qq, a)
        v[..., h:] = np.where(b >= qq, b - qq, b)
    return y * R.untwist % q if inverse else y


def ntt(x, R: Ring):
    """Forward negacyclic NTT over (..., k, n) (src/ring.py:408-430)."""
    x = np.asarray(x, dtype=U64)
    if R.jit:
        rows = np.ascontiguousarray(x).reshape(-1, R.n)
        return _rows_jit(rows, R.k, R.bitrev, R.twist, R._twist_sh, R._flat_f, R._flat_f_sh,
                         R.q[:, 0], False).reshape(x.shape)
    return _ntt_numpy(x, R, False)


def intt(x, R: Ring):
    """Inverse of :func:`ntt` (src/ring.py:433-453)."""
    x = np.asarray(x, dtype=U64)
    if R.jit:
        rows = np.ascontiguousarray(x).reshape(-1, R.n)
        return _rows_jit(rows, R.k, R.bitrev, R.untwist, R._untwist_sh, R._flat_i, R._flat_i_sh,
                         R.q[:, 0], True).reshape(x.shape)
    return _ntt_numpy(x, R, True)


def ntt_numpy(x, R: Ring):
    return _ntt_numpy(np.asarray(x, dtype=U64), R, False)


def intt_numpy(x, R: Ring):
    return _ntt_numpy(np.asarray(x, dtype=U64), R, True)


# ---------------------------------------------------------------------------
# CRT + centered gadget digits  (src/ring.py:456-495, src/he.py:323-367)

_M32 = U64(0xFFFFFFFF)


def crt_centered(x, R: Ring):
    """Centered CRT per coefficient -> (negative, magnitude as four 32-bit words, LSW first).

    X = sum_i y_i * (Q/q_i) with y_i = x_i * mhat_i mod q_i, reduced into [0, Q);
    negative = X > (Q-1)/2 and the magnitude is Q - X then (src/ring.py:456-495).
    Words are 32-bit so y_i * word < 2^59 and four partial sums stay below 2^64.
    """
    y = x * R.crt_mhat % R.q                       # (..., k, n)
    nw = (R.Q.bit_length() + 2 + 31) // 32 + 1      # words of k*Q plus one for carries
    acc = [np.zeros(y.shape[:-2] + (y.shape[-1],), dtype=U64) for _ in range(nw)]
    for i, m in enumerate(R.crt_m):
        yi = y[..., i, :]
        for w in range(nw):
            mw = (m >> (32 * w)) & 0xFFFFFFFF
            if mw:
                acc[w] = acc[w] + yi * U64(mw)
    words = []
    carry = np.zeros_like(acc[0])
    for w in range(nw):
        cur = acc[w] + carry
        words.append(cur & _M32)
        carry = cur >> U64(32)
    words = np.stack(words)                          # (nw, ..., n), each < 2^32
    # subtract multiples of Q: X < k*Q; descending powers of two times Q (src/ring.py:227-234)
    t = 1
    while t < R.k:
        t *= 2
    mults = []
    while t >= 1:
        mults.append(t * R.Q)
        t //= 2
    for mq in mults:
        words = _cond_sub(words, mq, nw)
    half = (R.Q - 1) // 2
    neg = _gt_const(words, half, nw)
    qminus = _sub_from_const(R.Q, words, nw)
    mag = np.where(neg[None], qminus, words)
    return neg, mag


def _const_words(c, nw):
    return [U64((c >> (32 * w)) & 0xFFFFFFFF) for w in range(nw)]


def _ge_const(words, c, nw):
    cw = _const_words(c, nw)
    ge = np.ones(words.shape[1:], dtype=bool)      # equal so far -> ge
    for w in range(nw):                             # from least to most significant
        gt = words[w] > cw[w]
        eq = words[w] == cw[w]
        ge = gt | (eq & ge)
    return ge


def _gt_const(words, c, nw):
    return _ge_const(words, c + 1, nw)


def _sub_words(a_words, b_words, nw):
    out, borrow = [], np.zeros(a_words[0].shape, dtype=U64)
    for w in range(nw):
        cur = a_words[w].astype(np.int64) - b_words[w].astype(np.int64) - borrow.astype(np.int64)
        borrow = (cur < 0).astype(U64)
        out.append((cur + (borrow.astype(np.int64) << 32)).astype(U64))
    return np.stack(out)


def _cond_sub(words, c, nw):
    ge = _ge_const(words, c, nw)
    cw = [np.full(words.shape[1:], v, dtype=U64) for v in _const_words(c, nw)]
    return np.where(ge[None], _sub_words(words, cw, nw), words)


def _sub_from_const(c, words, nw):
    cw = [np.full(words.shape[1:], v, dtype=U64) for v in _const_words(c, nw)]
    return _sub_words(cw, words, nw)


def gadget_digits(coeff, R: Ring, z_bits: int, ell: int):
    """Signed centered base-2^z_bits digits, (..., ell, n) int64 (src/he.py:346-362).

    Magnitude digits low to high; all but the last fold values > z/2 into
    (d - z, carry 1); the sign of the coefficient is applied to every digit.
    """
    neg, mag = crt_centered(coeff, R)
    if mag.shape[0] > 4 and np.any(mag[4:]):
        raise ValueError("magnitude exceeds 128 bits")
    z = 1 << z_bits
    zb, zmask = U64(z_bits), U64(z - 1)
    lo = mag[0] | (mag[1] << U64(32))
    hi = (mag[2] | (mag[3] << U64(32))) if mag.shape[0] > 3 else mag[2].copy()
    out = np.empty(neg.shape[:-1] + (ell, neg.shape[-1]), dtype=np.int64)
    for i in range(ell):
        raw = lo & zmask
        lo = (lo >> zb) | ((hi & zmask) << (U64(64) - zb))
        hi = hi >> zb
        d = raw.astype(np.int64)
        if i < ell - 1:
            adj = d > (z >> 1)
            d = np.where(adj, d - z, d)
            nlo = lo + adj.astype(U64)
            hi = hi + (nlo < lo).astype(U64)
            lo = nlo
        out[..., i, :] = np.where(neg, -d, d)
    return out


def lift(d, R: Ring):
    """Signed small ints (..., n) -> residues (..., k, n) (src/he.py:364-367)."""
    return (d[..., None, :] % R.q_i64).astype(U64)


# ---------------------------------------------------------------------------
# automorphism / monomials  (src/ring.py:643-673)

@lru_cache(maxsize=None)
def aut_perm(n: int, k_aut: int) -> np.ndarray:
    j = np.arange(n, dtype=np.int64)
    return (((2 * j + 1) * (k_aut % (2 * n))) % (2 * n) - 1) // 2


def monomial(R: Ring, e: int):
    j = np.arange(R.n, dtype=np.int64)
    return R.psi_pow[:, ((2 * j + 1) * (e % (2 * R.n))) % (2 * R.n)]


# ---------------------------------------------------------------------------
# tree geometry (src/planner.py:153-173)

def expansion_leaves(d0, d1, ell):
    return d0 + (d1.bit_length() - 1) * ell


def expand_stages(total):
    return math.ceil(math.log2(total)) if total > 1 else 0


# ---------------------------------------------------------------------------
# server primitives (src/planner.py:313-463)

def mac(digits_ntt, rows, R: Ring):
    """sum_i digits[i] * rows[i] over both ciphertext components (src/he.py:434-447).

    digits_ntt (..., L, k, n); rows (..., L, 2, k, n) -> (..., 2, k, n).
    Exact: products < 2^54, chunks of 512 products stay below 2^63.
    """
    q = R.q
    acc = None
    L = digits_ntt.shape[-3]
    for i in range(L):
        d = digits_ntt[..., i, None, :, :]
        term = d * rows[..., i, :, :, :] % q
        acc = term if acc is None else (acc + term) % q
    return acc


def subs_stage(state, ksks, k_aut, t, p: Params):
    """One ExpandQuery stage (src/planner.py:321-381): node c -> (c + Subs(c), X^-2^t (c - Subs(c))).

    state (B, C, 2, k, n); ksks (B, ell, 2, k, n) -> (B, 2C, 2, k, n).
    """
    R = p.ring
    perm = aut_perm(R.n, k_aut)
    aut = state[..., perm]
    a_coeff = intt(aut[:, :, 0], R)
    dig = gadget_digits(a_coeff, R, p.z_bits, p.ell)        # (B, C, ell, n)
    dn = ntt(lift(dig, R), R)                               # (B, C, ell, k, n)
    s = mac(dn, ksks[:, None], R)                           # (B, C, 2, k, n)
    s[:, :, 1] = (s[:, :, 1] + aut[:, :, 1]) % R.q
    mono = monomial(R, -(1 << t))
    out = np.empty(state.shape[:1] + (2 * state.shape[1],) + state.shape[2:], dtype=U64)
    C = state.shape[1]
    out[:, :C] = (state + s) % R.q
    out[:, C:] = mono * ((state + R.q - s) % R.q) % R.q
    return out


def expand(queries, evks, d0, d1, p: Params):
    """Full ExpandQuery (src/protocol.py:322-367): queries (B, 2, k, n), evks (B, stages, ell, 2, k, n)."""
    total = expansion_leaves(d0, d1, p.ell)
    state = np.asarray(queries, dtype=U64)[:, None]
    for t in range(expand_stages(total)):
        k_aut = p.n // (1 << t) + 1
        state = subs_stage(state, evks[:, t], k_aut, t, p)[:, :total]
    return state


def ext_product(cts, rows, p: Params):
    """cts (B, M, 2, k, n) ⊡ rows (B, 2ell, 2, k, n) (src/planner.py:384-435, src/he.py:468-484)."""
    R = p.ring
    coeff = intt(cts, R)                                    # (B, M, 2, k, n)
    dig = gadget_digits(coeff, R, p.z_bits, p.ell)          # (B, M, 2, ell, n)
    dn = ntt(lift(dig, R), R)                               # (B, M, 2, ell, k, n)
    B, M = cts.shape[:2]
    dn = dn.reshape(B, M, 2 * p.ell, R.k, R.n)              # a-digits then b-digits
    return mac(dn, rows[:, None], R)


def build_rgsw(col_cts, sk_rgsw, p: Params):
    """RGSW per column bit (src/protocol.py:383-409): rows[:ell] = col ⊡ RGSW(s), rows[ell:] = col.

    col_cts (B, bits*ell, 2, k, n), sk_rgsw (B, 2ell, 2, k, n) -> (B, bits, 2ell, 2, k, n).
    """
    B, M = col_cts.shape[:2]
    bits = M // p.ell
    out = np.empty((B, bits, 2 * p.ell) + col_cts.shape[2:], dtype=U64)
    if bits == 0:
        return out
    a_rows = ext_product(col_cts, sk_rgsw, p)
    for j in range(bits):
        out[:, j, :p.ell] = a_rows[:, j * p.ell:(j + 1) * p.ell]
        out[:, j, p.ell:] = col_cts[:, j * p.ell:(j + 1) * p.ell]
    return out


def rowsel(row_cts, db_pm, R: Ring):
    """Batched mod-q GEMM over p (src/protocol.py:448-501, src/layout.py:190-294).

    row_cts (B, d0, 2, k, n); db_pm (d1, d0, k*n) -> selected (B, d1, 2, k, n):
    out[b, j, c] = sum_i row_cts[b, i, c] * db[j, i] mod q.
    """
    B, d0 = row_cts.shape[:2]
    d1 = db_pm.shape[0]
    q = R.q
    a = row_cts.reshape(B, d0, 2, R.k, R.n)
    dbr = db_pm.reshape(d1, d0, R.k, R.n)
    out = np.zeros((B, d1, 2, R.k, R.n), dtype=U64)
    chunk = max(1, int((2**64 - 1) // (max(R.qs) - 1) ** 2))
    for j in range(d1):
        acc = np.zeros((B, 2, R.k, R.n), dtype=U64)
        for i0 in range(0, d0, chunk):
            part = np.zeros_like(acc)
            for i in range(i0, min(d0, i0 + chunk)):
                part += a[:, i] * dbr[j, i][None, None]
            acc = (acc + part % q) % q
        out[:, j] = acc
    return out


def coltor(selected, rgsws, p: Params):
    """Column tournament (src/protocol.py:542-573, src/planner.py:438-463), LSB first.

    selected (B, d1, 2, k, n); rgsws (B, bits, 2ell, 2, k, n) -> (B, 2, k, n).
    """
    R = p.ring
    s = selected
    for j in range(s.shape[1].bit_length() - 1):
        even, odd = s[:, 0::2], s[:, 1::2]
        diff = (odd + R.q - even) % R.q
        s = (even + ext_product(diff, rgsws[:, j], p)) % R.q
    return s[:, 0]


def answer_batch(queries, evks, sk_rgsws, db_pm, d0, d1, p: Params, stats=None):
    """Server pipeline (src/protocol.py:635-682) on raw arrays.

    queries (B, 2, k, n); evks (B, stages, ell, 2, k, n); sk_rgsws (B, 2ell, 2, k, n);
    db_pm (d1, d0, k*n) NTT-domain P-major.  Returns responses (B, 2, k, n).
    """
    import time
    t0 = time.perf_counter()
    leaves = expand(queries, evks, d0, d1, p)
    t1 = time.perf_counter()
    rg = build_rgsw(leaves[:, d0:], sk_rgsws, p)
    t2 = time.perf_counter()
    sel = rowsel(leaves[:, :d0], db_pm, p.ring)
    t3 = time.perf_counter()
    out = coltor(sel, rg, p)
    t4 = time.perf_counter()
    if stats is not None:
        for k_, v in (("ExpandQuery", t1 - t0), ("RgswAssembly", t2 - t1), ("RowSel", t3 - t2), ("ColTor", t4 - t3)):
            stats[k_] = stats.get(k_, 0.0) + v
    return out


# ---------------------------------------------------------------------------
# database encoding (src/protocol.py:102-153)

def encode_database(records, d0, d1, record_bytes, p: Params):
    """records (list of bytes, row-major r = i*d1 + j) -> (d1, d0, k*n) NTT-domain P-major."""
    R = p.ring
    width = p.plain_bits // 8
    half = p.P // 2
    m = np.zeros((d0 * d1, R.n), dtype=np.int64)
    for r, rec in enumerate(records):
        buf = rec.ljust(record_bytes, b"\x00")
        buf = buf.ljust(-(-len(buf) // width) * width, b"\x00")
        w = np.frombuffer(buf, dtype=f"<u{width}").astype(np.int64)
        m[r, :len(w)] = w
    m -= (m >= half) * p.P
    limbs = (m[:, None, :] % R.q_i64).astype(U64)
    nt = ntt(limbs, R)
    out = np.empty((d1, d0, R.k * R.n), dtype=U64)
    for r in range(d0 * d1):
        out[r % d1, r // d1] = nt[r].reshape(-1)
    return out


def decode_plain(m, record_bytes, p: Params) -> bytes:
    return m.astype(f"<u{p.plain_bits // 8}").tobytes()[:record_bytes]


# ---------------------------------------------------------------------------
# client side (keys, queries, decryption) — inputs/oracle checks only
# (src/he.py:220-316, 487-515; src/protocol.py:240-281)

@dataclass
class Client:
    p: Params
    s: np.ndarray               # secret, NTT domain (k, n)
    evks: np.ndarray            # (stages, ell, 2, k, n)
    sk_rgsw: np.ndarray         # (2ell, 2, k, n)


def _uniform(R, rng, shape=()):
    out = np.empty(shape + (R.k, R.n), dtype=U64)
    for i, q in enumerate(R.qs):
        out[..., i, :] = rng.integers(0, q, size=shape + (R.n,), dtype=np.uint64)
    return out


def _error(R, rng, bound):
    bits = rng.integers(0, 2, size=(2 * bound, R.n), dtype=np.int64)
    e = bits[:bound].sum(0) - bits[bound:].sum(0)
    return (e[None] % R.q_i64).astype(U64)


def encrypt_phase(p: Params, s, phase_ntt, rng):
    R = p.ring
    a = _uniform(R, rng)
    e = ntt(_error(R, rng, p.error_bound), R)
    b = (phase_ntt % R.q + R.q - a * s % R.q) % R.q
    return np.stack([a, (b + e) % R.q])


def client_keygen(p: Params, d0, d1, rng) -> Client:
    R = p.ring
    stages = expand_stages(expansion_leaves(d0, d1, p.ell))
    sc = rng.integers(-1, 2, size=R.n, dtype=np.int64)
    s = ntt((sc[None] % R.q_i64).astype(U64), R)
    zp = [np.array([pow(1 << p.z_bits, i, q) for q in R.qs], dtype=U64)[:, None] for i in range(p.ell)]
    evks = np.empty((stages, p.ell, 2, R.k, R.n), dtype=U64)
    for t in range(stages):
        s_aut = s[:, aut_perm(R.n, R.n // (1 << t) + 1)]
        for i in range(p.ell):
            evks[t, i] = encrypt_phase(p, s, zp[i] * s_aut % R.q, rng)
    rg = np.empty((2 * p.ell, 2, R.k, R.n), dtype=U64)
    ss = s * s % R.q
    for i in range(p.ell):  # a-digit rows first, then b-digit rows (src/he.py:494-500)
        rg[i] = encrypt_phase(p, s, zp[i] * ss % R.q, rng)
    for i in range(p.ell):
        rg[p.ell + i] = encrypt_phase(p, s, zp[i] * s % R.q, rng)
    return Client(p, s, evks, rg)


def client_query(c: Client, i_star, j_star, d0, d1, rng):
    p, R = c.p, c.p.ring
    total = expansion_leaves(d0, d1, p.ell)
    stages = expand_stages(total)
    pay = np.zeros((R.k, R.n), dtype=U64)
    for li, q in enumerate(R.qs):
        inv = pow(pow(2, stages, q), q - 2, q)
        pay[li, i_star] = p.delta % q * inv % q
        for bit in range(d1.bit_length() - 1):
            if (j_star >> bit) & 1:
                for dg in range(p.ell):
                    pay[li, d0 + bit * p.ell + dg] = pow(1 << p.z_bits, dg, q) * inv % q
    return encrypt_phase(p, c.s, ntt(pay, R), rng)


def decrypt(c: Client, ct):
    p, R = c.p, c.p.ring
    ph = intt((ct[1] + ct[0] * c.s % R.q) % R.q, R)
    neg, mag = crt_centered(ph, R)
    out = np.empty(R.n, dtype=U64)
    for j in range(R.n):
        v = sum(int(mag[w, j]) << (32 * w) for w in range(mag.shape[0]))
        v = -v if neg[j] else v
        out[j] = ((v * p.P + R.Q // 2) // R.Q) % p.P
    return out
