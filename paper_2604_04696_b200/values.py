"""Host-side value types and parameter sets of the GPIR server API.

These mirror the reference's containers so callers can switch imports
without code changes (src/ring.py:93-300, src/he.py:45-213,
src/protocol.py:38-237).  They only hold data; every computation on the server
path runs in libgpir.so.  The functions in `protocol` also accept the
reference's own objects (duck-typed on the same attribute names).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from functools import lru_cache
from typing import Sequence

import numpy as np

from .errors import InvalidArgument, InvalidState

U64 = np.uint64


class Domain(Enum):
    COEFF = "coeff"
    NTT = "ntt"


class LayoutKind(Enum):
    """Physical DB layouts of the reference (src/layout.py:39-41).  The GPU keeps
    its own brv P-major layout either way; the kind only tags the object."""

    P_MAJOR = "pmajor"
    TRANSPOSED = "transposed"


# ---------------------------------------------------------------------------
# primes and roots (setup only; src/ring.py:55-90, 239-254)

def is_prime(v: int) -> bool:
    if v < 2:
        return False
    wit = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for p in wit:
        if v % p == 0:
            return v == p
    d, s = v - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in wit:
        x = pow(a, d, v)
        if x in (1, v - 1):
            continue
        for _ in range(s - 1):
            x = x * x % v
            if x == v - 1:
                break
        else:
            return False
    return True


def find_two_n_root(q: int, two_n: int) -> int:
    if (q - 1) % two_n:
        raise InvalidArgument(f"q={q} is not 1 mod {two_n}")
    cof = (q - 1) // two_n
    for g in range(2, q):
        r = pow(g, cof, q)
        if pow(r, two_n // 2, q) == q - 1:
            return r
    raise InvalidArgument(f"no 2n-th root found mod {q}")


@dataclass(frozen=True)
class Modulus:
    q: int
    two_n_root: int


class RnsBasis:
    """Ordered RNS primes for ring degree n (src/ring.py:122-158)."""

    def __init__(self, n: int, moduli: Sequence[Modulus]):
        if n < 2 or n & (n - 1):
            raise InvalidArgument(f"ring degree must be a power of two >= 2, got {n}")
        if not moduli:
            raise InvalidArgument("need at least one modulus")
        qs = [m.q for m in moduli]
        if len(set(qs)) != len(qs):
            raise InvalidArgument("RNS primes must be pairwise distinct")
        for m in moduli:
            if not is_prime(m.q) or m.q.bit_length() > 31 or (m.q - 1) % (2 * n):
                raise InvalidArgument(f"{m.q} is not an NTT-friendly 31-bit prime for n={n}")
            if pow(m.two_n_root, n, m.q) != m.q - 1:
                raise InvalidArgument(f"root {m.two_n_root} does not have order {2 * n} mod {m.q}")
        self.n = n
        self.moduli = tuple(moduli)
        self.k = len(moduli)
        self.big_q = math.prod(qs)
        if (self.k * self.big_q).bit_length() > 128:
            raise InvalidArgument("k * Q must fit 128 bits")
        self.q_arr = np.array(qs, dtype=U64)
        self.q_col = self.q_arr[:, None]

    @classmethod
    def generate(cls, n: int, k: int, bits: int = 27) -> "RnsBasis":
        if bits > 31:
            raise InvalidArgument("primes must fit 32-bit storage")
        two_n = 2 * n
        moduli = []
        c = ((1 << bits) - 2) // two_n
        while len(moduli) < k and c > 0:
            q = c * two_n + 1
            if q.bit_length() <= bits and is_prime(q):
                moduli.append(Modulus(q, find_two_n_root(q, two_n)))
            c -= 1
        if len(moduli) < k:
            raise InvalidArgument(f"not enough {bits}-bit NTT primes for n={n}")
        return cls(n, moduli)

    def __repr__(self) -> str:
        return f"RnsBasis(n={self.n}, k={self.k}, Q~2^{self.big_q.bit_length() - 1})"


@lru_cache(maxsize=None)
def default_basis(n: int = 4096) -> RnsBasis:
    return RnsBasis.generate(n, 4, bits=27)


@dataclass(frozen=True)
class GadgetConfig:
    z_bits: int = 22
    ell: int = 5

    @property
    def z(self) -> int:
        return 1 << self.z_bits


@dataclass
class HeParams:
    """Ring, plaintext modulus P = 2^plain_bits and gadget (src/he.py:57-108)."""

    basis: RnsBasis
    plain_bits: int = 32
    gadget: GadgetConfig = field(default_factory=GadgetConfig)
    error_bound: int = 16

    def __post_init__(self):
        if self.plain_modulus >= self.basis.big_q:
            raise InvalidArgument("plaintext modulus must be smaller than Q")
        if self.basis.big_q // self.plain_modulus <= 1:
            raise InvalidArgument("Delta = floor(Q/P) must exceed 1")
        if self.gadget.z ** self.gadget.ell <= self.basis.big_q:
            raise InvalidArgument("gadget must satisfy z**ell > Q")

    @property
    def n(self) -> int:
        return self.basis.n

    @property
    def plain_modulus(self) -> int:
        return 1 << self.plain_bits

    @property
    def delta(self) -> int:
        return self.basis.big_q // self.plain_modulus

    @property
    def poly_bytes(self) -> int:
        return self.basis.k * self.basis.n * 4

    @property
    def ct_bytes(self) -> int:
        return 2 * self.poly_bytes


@lru_cache(maxsize=None)
def default_params(n: int = 4096) -> HeParams:
    return HeParams(default_basis(n))


def test_params(n: int = 256, k: int = 2, prime_bits: int = 27, plain_bits: int = 8,
                z_bits: int = 11, error_bound: int = 4) -> HeParams:
    basis = RnsBasis.generate(n, k, prime_bits)
    ell = 1
    while (1 << (z_bits * ell)) <= basis.big_q:
        ell += 1
    return HeParams(basis, plain_bits, GadgetConfig(z_bits, ell), error_bound)


test_params.__test__ = False  # not a pytest test


# ---------------------------------------------------------------------------
# ciphertext containers (src/he.py:137-213)

@dataclass
class RnsPoly:
    basis: RnsBasis
    limbs: np.ndarray
    domain: Domain

    def __post_init__(self):
        if self.limbs.shape != (self.basis.k, self.basis.n):
            raise InvalidArgument(f"limb matrix {self.limbs.shape} does not match basis")
        if self.limbs.dtype != U64:
            self.limbs = self.limbs.astype(U64)


@dataclass
class BfvCiphertext:
    a: RnsPoly
    b: RnsPoly

    @property
    def domain(self) -> Domain:
        return self.a.domain

    @property
    def basis(self) -> RnsBasis:
        return self.a.basis

    def raw(self) -> np.ndarray:
        return np.stack([self.a.limbs, self.b.limbs])


def ct_from_raw(raw: np.ndarray, basis: RnsBasis, domain: Domain = Domain.NTT) -> BfvCiphertext:
    return BfvCiphertext(RnsPoly(basis, np.ascontiguousarray(raw[0]), domain),
                         RnsPoly(basis, np.ascontiguousarray(raw[1]), domain))


@dataclass
class EvalKey:
    k_aut: int
    ksk: tuple
    gadget: GadgetConfig


@dataclass
class RgswCiphertext:
    rows: tuple
    gadget: GadgetConfig

    def raw(self) -> np.ndarray:
        return np.stack([r.raw() for r in self.rows])


# ---------------------------------------------------------------------------
# protocol containers (src/protocol.py:38-237)

@dataclass(frozen=True)
class DbConfig:
    d0: int
    d1: int
    record_bytes: int = 16384

    def __post_init__(self):
        if self.d0 < 1 or self.d1 < 1:
            raise InvalidArgument("database dimensions must be positive")
        if self.d1 & (self.d1 - 1):
            raise InvalidArgument("d1 must be a power of two (binary tournament)")
        if self.record_bytes < 1:
            raise InvalidArgument("record_bytes must be positive")

    @property
    def records(self) -> int:
        return self.d0 * self.d1

    def coords(self, flat_index: int) -> tuple[int, int]:
        if not 0 <= flat_index < self.records:
            raise InvalidArgument(f"record index {flat_index} out of range")
        return flat_index // self.d1, flat_index % self.d1


@dataclass
class ClientKeys:
    """Session material a client uploads once: one EvalKey per expansion stage and
    RGSW(s) (src/protocol.py:165-199)."""

    evks: list
    sk_rgsw: RgswCiphertext | None = None

    def __post_init__(self):
        self._by_kaut = {e.k_aut: e for e in self.evks}

    def evk_for(self, k_aut: int) -> EvalKey:
        evk = self._by_kaut.get(k_aut)
        if evk is None:
            raise InvalidState(f"no evaluation key for automorphism index {k_aut}")
        return evk

    def evk_raw(self, k_aut: int) -> np.ndarray:
        return np.stack([ct.raw() for ct in self.evk_for(k_aut).ksk])

    def sk_rgsw_raw(self) -> np.ndarray:
        if self.sk_rgsw is None:
            raise InvalidState("this key set has no RGSW of the secret (onion mode needs one)")
        return self.sk_rgsw.raw()


@dataclass
class ClientQuery:
    ct: BfvCiphertext
    client_id: int = 0
    seq: int = 0


@dataclass
class Response:
    ct: BfvCiphertext
    client_id: int = 0
    seq: int = 0
