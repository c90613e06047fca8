"""Generate golden vectors for the GPIR server path from the LIVE reference.

Run in the build container (the reference is not present on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/make_golden.py

It imports `latpir` from /root/reference/pkg/src and writes
`tests/golden/golden.json` (seeds, geometry, SHA-256 digests of every phase's
output) and `tests/golden/vectors.npz` (small explicit vectors: NTT, digits,
toy responses).  Inputs are regenerated from seeds by the oracle's client,
which consumes the numpy RNG in exactly the reference's order
(src/he.py:220-271, src/protocol.py:246-281), so fixtures stay small; the
digests of the reference's keys and queries are stored too, so a drift in
that replay is caught before any server output is compared.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from latpir import he, planner, protocol, ring  # noqa: E402
from latpir.planner import ExecMode  # noqa: E402


def digest(a) -> str:
    a = np.asarray(a)
    return hashlib.sha256(np.ascontiguousarray(a.astype("<u4")).tobytes()).hexdigest()


def make_params(spec):
    if spec["profile"] == "default":
        basis = ring.default_basis(spec.get("n", 4096))
        return he.HeParams(basis, spec.get("plain_bits", 32))
    kw = {k: spec[k] for k in ("n", "k", "prime_bits", "plain_bits", "z_bits", "error_bound") if k in spec}
    return he.test_params(**kw)


def pipeline_case(name, spec, d0, d1, rec_bytes, db_seed, clients, queries, mode=None):
    """clients: list of (client_id, seed); queries: list of (client_id, i, j)."""
    params = make_params(spec)
    cfg = protocol.DbConfig(d0, d1, rec_bytes)
    rng = np.random.default_rng(db_seed)
    records = [rng.integers(0, 256, size=rec_bytes, dtype=np.uint8).tobytes() for _ in range(cfg.records)]
    db = protocol.encode_database(records, cfg, params)
    sessions = {}
    for cid, seed in clients:
        crng = np.random.default_rng(seed)
        sessions[cid] = (protocol.ClientSession.create(params, cfg, crng, client_id=cid), crng)
    qs = []
    for cid, i, j in queries:
        s, crng = sessions[cid]
        qs.append(s.gen_query(i, j, crng))
    keys = {cid: s.keys for cid, (s, _) in sessions.items()}
    klist = [keys[q.client_id] for q in qs]
    expanded = protocol.expand_query_batch(qs, klist, cfg, params, mode=mode or ExecMode.OPERATION_LEVEL)
    leaves = np.stack([np.stack([ct.raw() for ct in ex.row_cts + ex.col_cts]) for ex in expanded])
    rgsws = [protocol.build_rgsw_from_expanded(ex.col_cts, k, params) for ex, k in zip(expanded, klist)]
    rg = np.stack([np.stack([r.raw() for r in per]) if per else np.zeros((0,)) for per in rgsws]) if rgsws[0] else None
    in0 = protocol._expanded_to_in0(expanded, params)
    out_pm, _ = protocol.row_select_raw(in0, db, params)
    selected = protocol._out_to_stack(out_pm, params)
    resp = protocol.answer_batch(qs, keys, db, params)
    final = np.stack([r.ct.raw() for r in resp])
    dec_ok = [sessions[q.client_id][0].decode(r) == records[i * d1 + j] for q, r, (_, i, j) in zip(qs, resp, queries)]
    case = {
        "name": name, "params": spec, "d0": d0, "d1": d1, "record_bytes": rec_bytes, "db_seed": db_seed,
        "clients": clients, "queries": queries,
        "n": params.n, "k": params.basis.k, "qs": [m.q for m in params.basis.moduli],
        "psis": [m.two_n_root for m in params.basis.moduli], "ell": params.gadget.ell,
        "z_bits": params.gadget.z_bits,
        "digest": {
            "db": digest(db.data),
            "evks": {str(cid): digest(np.stack([np.stack([c.raw() for c in e.ksk]) for e in s.keys.evks]))
                     for cid, (s, _) in sessions.items()},
            "sk_rgsw": {str(cid): digest(s.keys.sk_rgsw.raw()) for cid, (s, _) in sessions.items()},
            "queries": digest(np.stack([q.ct.raw() for q in qs])),
            "leaves": digest(leaves),
            "rgsw": digest(rg) if rg is not None else None,
            "selected": digest(selected),
            "responses": digest(final),
        },
        "decrypt_ok": dec_ok,
    }
    return case, final


def main():
    os.makedirs(OUT, exist_ok=True)
    vec = {}
    cases = []

    # --- transform / digit KATs on the tiny and production rings -------------------
    for tag, params in (("tiny", he.test_params(n=64, k=2, prime_bits=20, plain_bits=8, z_bits=7, error_bound=2)),
                        ("proto", he.test_params()),
                        ("prod", he.default_params())):
        b = params.basis
        rng = np.random.default_rng(101)
        x = np.stack([ring.sample_uniform(b, b.n, rng).limbs for _ in range(3)])
        vec[f"{tag}_ntt_in"] = x.astype(np.uint32)
        vec[f"{tag}_ntt_out"] = ring.ntt_raw(x, b).astype(np.uint32)
        vec[f"{tag}_intt_out"] = ring.intt_raw(x, b).astype(np.uint32)
        ex = he.DigitExtractor(x, b, params.gadget)
        vec[f"{tag}_digits"] = np.stack([ex.next_signed() for _ in range(params.gadget.ell)], axis=1).astype(np.int32)
        vec[f"{tag}_qs"] = np.array([m.q for m in b.moduli], dtype=np.uint64)
        vec[f"{tag}_psis"] = np.array([m.two_n_root for m in b.moduli], dtype=np.uint64)
        # one subs and one external product on random material
        st = np.stack([np.stack([ring.sample_uniform(b, b.n, rng).limbs for _ in range(2)]) for _ in range(2)])[None]
        ks = np.stack([np.stack([ring.sample_uniform(b, b.n, rng).limbs for _ in range(2)])
                       for _ in range(params.gadget.ell)])[None]
        t = 1
        mono = ring.monomial_ntt(b, -(1 << t))
        out = planner.expand_stage(st, ks, b.n // (1 << t) + 1, mono, b, params.gadget, ExecMode.OPERATION_LEVEL)
        vec[f"{tag}_subs_in"] = st.astype(np.uint32)
        vec[f"{tag}_subs_ksk"] = ks.astype(np.uint32)
        vec[f"{tag}_subs_out"] = out.astype(np.uint32)
        rows = np.stack([np.stack([ring.sample_uniform(b, b.n, rng).limbs for _ in range(2)])
                         for _ in range(2 * params.gadget.ell)])[None]
        xp = planner.external_product_batch(st, rows, b, params.gadget, ExecMode.STAGE_LEVEL)
        vec[f"{tag}_xp_rows"] = rows.astype(np.uint32)
        vec[f"{tag}_xp_out"] = xp.astype(np.uint32)
        # a rowsel GEMM
        pflat = b.k * b.n
        in0 = rng.integers(0, 1 << 26, size=(4, 5, pflat), dtype=np.uint64) % np.repeat(b.q_arr, b.n)
        dbt = rng.integers(0, 1 << 26, size=(2, 5, pflat), dtype=np.uint64) % np.repeat(b.q_arr, b.n)
        qp = np.repeat(b.q_arr, b.n)
        from latpir import layout
        vec[f"{tag}_gemm_a"] = in0.astype(np.uint32)
        vec[f"{tag}_gemm_b"] = dbt.astype(np.uint32)
        vec[f"{tag}_gemm_out"] = layout.gemm_pmajor_tiled(in0, dbt, qp, layout.auto_tile(4, 2, 5, pflat, pmajor=True)).astype(np.uint32)
        print("kat", tag, "done", flush=True)

    # --- full pipeline cases ------------------------------------------------------------
    proto = {"profile": "test"}
    c, final = pipeline_case("proto_8x8", proto, 8, 8, 64, 1234, [[0, 11], [1, 12]],
                             [[0, 3, 5], [1, 0, 0], [0, 7, 7]])
    vec["proto_8x8_responses"] = final.astype(np.uint32)
    cases.append(c)
    print("case", c["name"], c["decrypt_ok"], flush=True)
    c, final = pipeline_case("proto_5x1", proto, 5, 1, 16, 77, [[4, 21]], [[4, 2, 0], [4, 4, 0]])
    vec["proto_5x1_responses"] = final.astype(np.uint32)
    cases.append(c)
    print("case", c["name"], c["decrypt_ok"], flush=True)
    c, final = pipeline_case("prod_4x4", {"profile": "default"}, 4, 4, 1024, 99, [[7, 31]], [[7, 1, 2], [7, 3, 3]])
    vec["prod_4x4_responses_head"] = final[..., :64].astype(np.uint32)
    cases.append(c)
    print("case", c["name"], c["decrypt_ok"], flush=True)
    c, _ = pipeline_case("prod_16x16", {"profile": "default"}, 16, 16, 16384, 20260811, [[1, 5]],
                         [[1, 9, 13], [1, 0, 15]])
    cases.append(c)
    print("case", c["name"], c["decrypt_ok"], flush=True)
    c, _ = pipeline_case("prod_p16_256x2", {"profile": "default", "plain_bits": 16}, 256, 2, 8192, 314,
                         [[2, 9]], [[2, 255, 1]])
    cases.append(c)
    print("case", c["name"], c["decrypt_ok"], flush=True)

    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump({"generator": "tools/make_golden.py", "reference": "latpir (/root/reference/pkg)",
                   "cases": cases}, fh, indent=1)
    np.savez_compressed(os.path.join(OUT, "vectors.npz"), **vec)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
