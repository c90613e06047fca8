"""Digit-extraction boundary vectors from the LIVE reference (build container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/make_digit_golden.py

Crafted centered coefficients on the production ring (N=4096, k=4 primes of
27 bits, Q ~ 2^108, z = 2^22, ell = 5) that hit every branch of the
reference's sign-magnitude carry rule (src/latpir/he.py:323-367): a raw digit
equal to z/2 (stays positive), z/2 + 1 (carries), carry chains through all
ell digits, the extremes 0, +-1, +-(Q-1)/2, and digit patterns drawn from
{0, 1, z/2 - 1, z/2, z/2 + 1, z - 1} at every position with both signs.
The reference's DigitExtractor (CRT via crt_to_words, then next_signed) and
its scalar oracle centered_digits_int produce the expected digits; both must
agree or the script aborts.  Output: tests/golden/digits_boundary.npz with
`coeff` (polys, k, n) uint32 residues and `digits` (polys, ell, n) int32.
"""
from __future__ import annotations

import itertools
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden", "digits_boundary.npz")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from latpir import he, ring  # noqa: E402


def crafted(Q: int, z: int, ell: int, n: int, rng) -> list[int]:
    half = (Q - 1) // 2
    vals = [0, 1, -1, half, -half, half - 1, -(half - 1), z // 2, -(z // 2), z // 2 + 1, -(z // 2 + 1)]
    for j in range(ell):
        for r in (z // 2 - 1, z // 2, z // 2 + 1, z - 1):
            vals += [r * z**j, -r * z**j, r * z**j + z**j - 1, z**(j + 1) - 1, z**j]
    # carry chains: every low digit > z/2 (carries ripple through all ell - 1 of them), or == z/2 (no carry)
    for r in (z // 2 + 1, z - 1, z // 2):
        for top in (0, 1, 5):
            m = sum(r * z**j for j in range(ell - 1)) + top * z**(ell - 1)
            vals += [m, -m]
    # digit patterns at every position (top digit bounded so |c| <= (Q-1)/2)
    pick = [0, 1, z // 2 - 1, z // 2, z // 2 + 1, z - 1]
    top_max = half >> ((ell - 1) * 22)
    for combo in itertools.product(pick, repeat=ell - 1):
        for top in (0, 1, top_max // 2, top_max - 1):
            m = sum(d * z**j for j, d in enumerate(combo)) + top * z**(ell - 1)
            if m <= half:
                vals.append(int(m) if rng.random() < 0.5 else -int(m))
    vals = [v for v in vals if abs(v) <= half]
    pad = (-len(vals)) % n
    vals += [int(rng.integers(-(1 << 62), 1 << 62)) * int(rng.integers(1, 1 << 40)) % (2 * half + 1) - half
             for _ in range(pad)]
    return vals


def main() -> None:
    basis = ring.default_basis(4096)
    params = he.HeParams(basis, 32)
    g = params.gadget
    z, ell, n = g.z, g.ell, basis.n
    qs = [int(m.q) for m in basis.moduli]
    Q = 1
    for q in qs:
        Q *= q
    rng = np.random.default_rng(20261017)
    vals = crafted(Q, z, ell, n, rng)
    polys = len(vals) // n
    coeff = np.zeros((polys, len(qs), n), dtype=np.uint64)
    for idx, v in enumerate(vals):
        for i, q in enumerate(qs):
            coeff[idx // n, i, idx % n] = v % q
    ex = he.DigitExtractor(coeff, basis, g)
    digits = np.stack([ex.next_signed() for _ in range(ell)], axis=1)  # (polys, ell, n)
    for idx, v in enumerate(vals):  # the reference's two implementations must agree
        want = he.centered_digits_int(v, Q, z, ell)
        got = [int(digits[idx // n, j, idx % n]) for j in range(ell)]
        assert got == want, (v, got, want)
    np.savez_compressed(OUT, coeff=coeff.astype(np.uint32), digits=digits.astype(np.int32))
    print(f"wrote {OUT}: {len(vals)} coefficients in {polys} polys")


if __name__ == "__main__":
    main()
