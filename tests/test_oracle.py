"""Pin the CPU oracle against the golden vectors produced by the live reference
(tools/make_golden.py).  CPU only."""
import os

import numpy as np
import pytest

from oracle import gpir_oracle as O
from tests.helpers import digest, oracle_params, rebuild_case

PROFILES = {
    "tiny": dict(n=64, k=2, prime_bits=20, plain_bits=8, z_bits=7, error_bound=2),
    "proto": dict(),
    "prod": None,
}


def _params(tag):
    return O.default_params() if PROFILES[tag] is None else O.test_params(**PROFILES[tag])


@pytest.mark.parametrize("tag", list(PROFILES))
def test_ring_matches_reference_primes(golden, tag):
    _, vec = golden
    p = _params(tag)
    assert p.ring.qs == [int(v) for v in vec[f"{tag}_qs"]]
    assert p.ring.psis == [int(v) for v in vec[f"{tag}_psis"]]


@pytest.mark.parametrize("tag", list(PROFILES))
@pytest.mark.parametrize("path", ["jit", "numpy"])
def test_ntt_golden(golden, tag, path):
    _, vec = golden
    R = _params(tag).ring
    x = vec[f"{tag}_ntt_in"].astype(np.uint64)
    f, i = (O.ntt, O.intt) if path == "jit" else (O.ntt_numpy, O.intt_numpy)
    assert np.array_equal(f(x, R), vec[f"{tag}_ntt_out"])
    assert np.array_equal(i(x, R), vec[f"{tag}_intt_out"])
    assert np.array_equal(i(f(x, R), R), x)


@pytest.mark.parametrize("tag", list(PROFILES))
def test_digits_golden(golden, tag):
    _, vec = golden
    p = _params(tag)
    x = vec[f"{tag}_ntt_in"].astype(np.uint64)
    d = O.gadget_digits(x, p.ring, p.z_bits, p.ell)
    assert np.array_equal(d, vec[f"{tag}_digits"])
    # recomposition law (src/he.py:14-16): sum d_i z^i == x mod every q
    acc = np.zeros_like(x)
    for i in range(p.ell):
        zi = np.array([pow(1 << p.z_bits, i, q) for q in p.ring.qs], dtype=np.uint64)[:, None]
        acc = (acc + zi * O.lift(d[..., i, :], p.ring)) % p.ring.q
    assert np.array_equal(acc, x)


def test_expansion_geometry():
    # src/planner.py:153-159: leaves = d0 + log2(d1)*ell, stages = ceil(log2(leaves))
    assert O.expansion_leaves(256, 64, 5) == 286 and O.expand_stages(286) == 9
    assert O.expansion_leaves(16, 16, 5) == 36 and O.expand_stages(36) == 6
    assert O.expand_stages(1) == 0
    assert list(O.aut_perm(4096, 4097)[:4]) == [2048, 2049, 2050, 2051]
    assert list(O.aut_perm(4096, 17)[:4]) == [8, 25, 42, 59]


@pytest.mark.parametrize("tag", list(PROFILES))
def test_subs_and_external_product_golden(golden, tag):
    _, vec = golden
    p = _params(tag)
    st = vec[f"{tag}_subs_in"].astype(np.uint64)
    ks = vec[f"{tag}_subs_ksk"].astype(np.uint64)
    out = O.subs_stage(st, ks, p.n // 2 + 1, 1, p)
    assert np.array_equal(out, vec[f"{tag}_subs_out"])
    rows = vec[f"{tag}_xp_rows"].astype(np.uint64)
    assert np.array_equal(O.ext_product(st, rows, p), vec[f"{tag}_xp_out"])


@pytest.mark.parametrize("tag", list(PROFILES))
def test_rowsel_golden(golden, tag):
    _, vec = golden
    p = _params(tag)
    a = vec[f"{tag}_gemm_a"].astype(np.uint64)    # (m=4, k=5, p)
    d = vec[f"{tag}_gemm_b"].astype(np.uint64)    # (n=2, k=5, p)
    R = p.ring
    rows = a.reshape(2, 2, 5, R.k, R.n).transpose(0, 2, 1, 3, 4)   # (B, d0, comp, k, n), m = 2b + comp
    sel = O.rowsel(rows, d, R)                                      # (B, d1, 2, k, n)
    want = vec[f"{tag}_gemm_out"].reshape(2, 2, 2, R.k, R.n).transpose(0, 2, 1, 3, 4)
    assert np.array_equal(sel, want)


CASES_FAST = ["proto_8x8", "proto_5x1", "prod_4x4"]


@pytest.mark.parametrize("name", CASES_FAST + ["prod_16x16"])
def test_pipeline_golden(golden, name):
    cases, vec = golden
    case = cases[name]
    p, records, clients, queries = rebuild_case(case)
    dg = case["digest"]
    for cid, c in clients.items():
        assert digest(c.evks) == dg["evks"][str(cid)], "client replay drifted from the reference RNG order"
        assert digest(c.sk_rgsw) == dg["sk_rgsw"][str(cid)]
    assert digest(np.stack(queries)) == dg["queries"]
    db = O.encode_database(records, case["d0"], case["d1"], case["record_bytes"], p)
    assert digest(db) == dg["db"]
    cids = [q[0] for q in case["queries"]]
    evks = np.stack([clients[c].evks for c in cids])
    rg = np.stack([clients[c].sk_rgsw for c in cids])
    leaves = O.expand(np.stack(queries), evks, case["d0"], case["d1"], p)
    assert digest(leaves) == dg["leaves"]
    rgsw = O.build_rgsw(leaves[:, case["d0"]:], rg, p)
    if dg["rgsw"] is not None:
        assert digest(rgsw) == dg["rgsw"]
    sel = O.rowsel(leaves[:, :case["d0"]], db, p.ring)
    assert digest(sel) == dg["selected"]
    out = O.coltor(sel, rgsw, p)
    assert digest(out) == dg["responses"]
    if f"{name}_responses" in vec.files:
        assert np.array_equal(out, vec[f"{name}_responses"])
    for (cid, i, j), ct in zip(case["queries"], out):
        m = O.decrypt(clients[cid], ct)
        assert O.decode_plain(m, case["record_bytes"], p) == records[i * case["d1"] + j]


def test_digits_boundary_vectors():
    """Digit-extraction boundary vectors made by the live reference's DigitExtractor and
    centered_digits_int (tools/make_digit_golden.py): raw digits at z/2 and z/2 + 1 at every
    position, carry chains through all ell digits, 0, +-1, +-(Q-1)/2."""
    v = np.load(os.path.join(os.path.dirname(__file__), "golden", "digits_boundary.npz"))
    p = O.default_params()
    got = O.gadget_digits(v["coeff"].astype(np.uint64), p.ring, p.z_bits, p.ell)
    assert np.array_equal(got, v["digits"].astype(np.int64))
