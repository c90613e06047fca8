"""Wire-format golden fixtures from the LIVE reference (src/wire.py).

Run in the build container (the reference does not travel to the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/make_wire_golden.py

Writes tests/golden/wire.npz:
  * query_{i} / response_{i}: messages serialised by latpir.wire from a real
    client session on the test ring (n=256, k=2), plus the decoded arrays;
  * evkset: a full key-set upload for a 8x8 DB and its decoded evks / RGSW;
  * bad_*: malformed messages with the reference's ParseError message and offset;
  * gpdb_{pmajor,transposed}: DB container images written by latpir.wire.save_database
    (4x2 DB) and the P-major tensor load_database returns for them.
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden", "wire.npz")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from latpir import he, protocol, wire  # noqa: E402
from latpir.errors import ParseError  # noqa: E402
from latpir.layout import LayoutKind  # noqa: E402


def perr(fn, *a):
    try:
        fn(*a)
    except ParseError as exc:
        return str(exc), int(exc.offset)
    raise AssertionError("no ParseError")


def main():
    params = he.test_params()
    basis = params.basis
    cfg = protocol.DbConfig(8, 8, 32)
    rng = np.random.default_rng(7)
    sess = protocol.ClientSession.create(params, cfg, rng, client_id=3)
    out: dict = {}
    meta: dict = {"n": basis.n, "k": basis.k, "qs": [m.q for m in basis.moduli], "z_bits": params.gadget.z_bits,
                  "ell": params.gadget.ell, "plain_bits": params.plain_bits, "bad": {}}
    for i, (r, c) in enumerate([(0, 0), (5, 3), (7, 7)]):
        q = sess.gen_query(r, c, rng)
        q = protocol.ClientQuery(q.ct, q.client_id, 100 + i)
        msg = wire.serialize_query(q)
        out[f"query_{i}"] = np.frombuffer(msg, np.uint8)
        out[f"query_{i}_ct"] = np.stack([q.ct.a.limbs, q.ct.b.limbs]).astype(np.uint32)
        out[f"query_{i}_route"] = np.array([q.client_id, q.seq], np.uint64)
        resp = protocol.Response(q.ct, q.client_id, q.seq)  # any NTT ct exercises the codec
        out[f"response_{i}"] = np.frombuffer(wire.serialize_response(resp), np.uint8)
    evk = wire.serialize_evkset(3, sess.keys)
    out["evkset"] = np.frombuffer(evk, np.uint8)
    stages = protocol.expansion_stage_count(cfg, params)
    meta["evk_stages"] = stages
    out["evkset_evks"] = np.stack([sess.keys.evk_raw(basis.n // (1 << t) + 1) for t in range(stages)]).astype(np.uint32)
    out["evkset_rgsw"] = sess.keys.sk_rgsw_raw().astype(np.uint32)

    q0 = bytes(out["query_0"])
    bad = {
        "short_header": q0[:10],
        "bad_magic": b"XPIR" + q0[4:],
        "bad_version": q0[:4] + (7).to_bytes(2, "little") + q0[6:],
        "length_mismatch": q0 + b"\x00",
        "wrong_kind": wire.serialize_response(protocol.Response(sess.gen_query(1, 1, rng).ct, 3, 1)),
        "bad_echo": q0[:27] + (basis.n * 2).to_bytes(4, "little") + q0[31:],
        "truncated_ct": q0[:15] + (len(q0) - 15 - 100).to_bytes(8, "little")[:8] + q0[23:-100],
        "trailing": q0[:7] + (len(q0) - 15 + 4).to_bytes(8, "little") + q0[15:] + b"\x00" * 4,
    }
    for name, b in bad.items():
        out[f"bad_{name}"] = np.frombuffer(b, np.uint8)
        meta["bad"][name] = perr(wire.deserialize_query, b, basis)

    # DB containers
    recs = [rng.integers(0, 256, size=cfg.record_bytes, dtype=np.uint8).tobytes() for _ in range(4 * 2)]
    small = protocol.DbConfig(4, 2, cfg.record_bytes)
    db = protocol.encode_database(recs, small, params)
    with tempfile.TemporaryDirectory() as td:
        for kind in (LayoutKind.P_MAJOR, LayoutKind.TRANSPOSED):
            path = os.path.join(td, "db.gpdb")
            wire.save_database(path, db.to_layout(kind))
            img = open(path, "rb").read()
            tag = "pmajor" if kind is LayoutKind.P_MAJOR else "transposed"
            out[f"gpdb_{tag}"] = np.frombuffer(img, np.uint8)
            ldb, _ = wire.load_database(path, params)
            out[f"gpdb_{tag}_data"] = ldb.to_layout(LayoutKind.P_MAJOR).data.astype(np.uint32)
        meta["gpdb_geometry"] = [small.d0, small.d1, small.record_bytes]
        img = bytes(out["gpdb_pmajor"])
        meta["gpdb_bad"] = {}
        for name, b in {"short": img[:20], "magic": b"XPDB" + img[4:], "truncated": img[:-8]}.items():
            path = os.path.join(td, name)
            open(path, "wb").write(b)
            meta["gpdb_bad"][name] = perr(wire.load_database, path, params)
            out[f"gpdb_bad_{name}"] = np.frombuffer(b, np.uint8)
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, sorted(meta["bad"].items())[:3])


if __name__ == "__main__":
    main()
