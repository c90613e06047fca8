"""Shared test helpers: rebuild golden-case inputs from seeds with the oracle client."""
from __future__ import annotations

import hashlib

import numpy as np

from oracle import gpir_oracle as O


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a).astype("<u4")).tobytes()).hexdigest()


def oracle_params(spec) -> O.Params:
    if spec["profile"] == "default":
        return O.default_params(spec.get("n", 4096), spec.get("plain_bits", 32))
    kw = {k: spec[k] for k in ("n", "k", "prime_bits", "plain_bits", "z_bits", "error_bound") if k in spec}
    return O.test_params(**kw)


def rebuild_case(case):
    """Regenerate records, client material and queries exactly as tools/make_golden.py did
    (the oracle client consumes the RNG in the reference's order)."""
    p = oracle_params(case["params"])
    d0, d1, rb = case["d0"], case["d1"], case["record_bytes"]
    rng = np.random.default_rng(case["db_seed"])
    records = [rng.integers(0, 256, size=rb, dtype=np.uint8).tobytes() for _ in range(d0 * d1)]
    clients, rngs = {}, {}
    for cid, seed in case["clients"]:
        r = np.random.default_rng(seed)
        clients[cid] = O.client_keygen(p, d0, d1, r)
        rngs[cid] = r
    queries = []
    for cid, i, j in case["queries"]:
        queries.append(O.client_query(clients[cid], i, j, d0, d1, rngs[cid]))
    return p, records, clients, queries


def to_api(params_o: O.Params):
    """The package's HeParams for an oracle parameter set."""
    import paper_2604_04696_b200 as G
    R = params_o.ring
    basis = G.RnsBasis(R.n, [G.Modulus(q, psi) for q, psi in zip(R.qs, R.psis)])
    return G.HeParams(basis, params_o.plain_bits, G.GadgetConfig(params_o.z_bits, params_o.ell),
                      params_o.error_bound)


def api_keys(params, client: O.Client):
    """ClientKeys (package types) from oracle key arrays."""
    import paper_2604_04696_b200 as G
    b, g = params.basis, params.gadget
    n = b.n
    evks = []
    for t in range(client.evks.shape[0]):
        ksk = tuple(G.ct_from_raw(client.evks[t, i], b) for i in range(g.ell))
        evks.append(G.EvalKey(n // (1 << t) + 1, ksk, g))
    rg = G.RgswCiphertext(tuple(G.ct_from_raw(client.sk_rgsw[r], b) for r in range(2 * g.ell)), g)
    return G.ClientKeys(evks, rg)


def api_query(params, ct, client_id=0, seq=0):
    import paper_2604_04696_b200 as G
    return G.ClientQuery(G.ct_from_raw(ct, params.basis), client_id, seq)
