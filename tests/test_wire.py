"""Wire codec, DB container and batch collector against
fixtures written by the live reference (tools/make_wire_golden.py).

The codec is host code in libgpir.so, so these run without a GPU; the GPDB
loader and the end-to-end collector run on the GPU (marked)."""
import json
import os
import tempfile
import threading

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def W():
    z = np.load(os.path.join(HERE, "golden", "wire.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


@pytest.fixture(scope="module")
def params(W):
    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200.values import find_two_n_root

    _, m = W
    basis = G.RnsBasis(m["n"], [G.Modulus(q, find_two_n_root(q, 2 * m["n"])) for q in m["qs"]])
    return G.HeParams(basis, m["plain_bits"], G.GadgetConfig(m["z_bits"], m["ell"]), 4)


def test_decode_queries_matches_reference(W, params):
    from paper_2604_04696_b200 import wire
    z, m = W
    msgs = [bytes(z[f"query_{i}"]) for i in range(3)]
    arr, ids, seqs = wire.decode_queries(msgs, m["n"], m["k"])
    for i in range(3):
        assert np.array_equal(arr[i], z[f"query_{i}_ct"])
        assert [int(ids[i]), int(seqs[i])] == [int(v) for v in z[f"query_{i}_route"]]
    q = wire.deserialize_query(msgs[1], params.basis)
    assert (q.client_id, q.seq) == (3, 101)
    assert np.array_equal(q.ct.raw(), z["query_1_ct"])
    assert wire.serialize_query(q) == msgs[1]


def test_encode_responses_matches_reference(W, params):
    from paper_2604_04696_b200 import wire
    z, m = W
    raw = np.stack([z[f"query_{i}_ct"] for i in range(3)])
    routes = np.stack([z[f"query_{i}_route"] for i in range(3)])
    msgs = wire.encode_responses(raw, routes[:, 0], routes[:, 1])
    for i in range(3):
        assert msgs[i] == bytes(z[f"response_{i}"])
        r = wire.deserialize_response(msgs[i], params.basis)
        assert np.array_equal(r.ct.raw(), raw[i]) and (r.client_id, r.seq) == tuple(int(v) for v in routes[i])


@pytest.mark.parametrize("name", ["short_header", "bad_magic", "bad_version", "length_mismatch", "wrong_kind",
                                  "bad_echo", "truncated_ct", "trailing"])
def test_parse_errors_match_reference(W, params, name):
    from paper_2604_04696_b200 import ParseError, wire
    z, m = W
    msg, off = m["bad"][name]
    with pytest.raises(ParseError) as ei:
        wire.deserialize_query(bytes(z[f"bad_{name}"]), params.basis)
    assert str(ei.value) == msg and ei.value.offset == off


def test_batch_decode_reports_bad_index(W):
    from paper_2604_04696_b200 import ParseError, wire
    z, m = W
    msgs = [bytes(z["query_0"]), bytes(z["query_1"]), bytes(z["bad_bad_echo"])]
    with pytest.raises(ParseError) as ei:
        wire.decode_queries(msgs, m["n"], m["k"])
    assert ei.value.index == 2


def test_evkset_matches_reference(W, params):
    from paper_2604_04696_b200 import wire
    z, m = W
    cid, keys = wire.decode_evkset(bytes(z["evkset"]), params, m["evk_stages"])
    assert cid == 3
    assert np.array_equal(keys.evks, z["evkset_evks"])
    assert np.array_equal(keys.sk_rgsw_raw(), z["evkset_rgsw"])
    for t in range(m["evk_stages"]):
        assert np.array_equal(keys.evk_raw(m["n"] // (1 << t) + 1), z["evkset_evks"][t])


def _stub_answer(monkeypatch, calls):
    from paper_2604_04696_b200 import protocol

    def fake(qarr, ids, keys, db, params, **kw):
        calls.append((qarr.shape[0], [int(i) for i in ids]))
        return qarr.copy()  # echo: response ct = query ct

    monkeypatch.setattr(protocol, "answer_raw", fake)


class _DB:
    def __init__(self, d0, d1, rb):
        from paper_2604_04696_b200 import DbConfig
        self.config = DbConfig(d0, d1, rb)


def test_collector_batches_and_replies(W, params, monkeypatch):
    """batch_max cut, arrival-order replies, malformed messages answered with
    error code 1 while the rest of the batch is served (src/server.py:222-292)."""
    from paper_2604_04696_b200 import server, wire
    z, m = W
    calls = []
    _stub_answer(monkeypatch, calls)
    col = server.BatchCollector(_DB(8, 8, 32), params, server.CollectorConfig(batch_max=2, batch_wait_ms=5))
    got = {}
    done = threading.Event()

    def reply_for(i):
        def r(b):
            got[i] = b
            if len(got) == 4:
                done.set()
        return r

    msgs = [bytes(z["query_0"]), bytes(z["bad_trailing"]), bytes(z["query_1"]), bytes(z["query_2"])]
    with col:
        for i, msg in enumerate(msgs):
            col.handle_message(msg, reply_for(i))
        assert done.wait(10)
    assert all(n <= 2 for n, _ in calls) and sum(n for n, _ in calls) == 3
    code, text = server.deserialize_error(got[1])
    assert code == 1 and text == m["bad"]["trailing"][0]
    for i, qi in ((0, 0), (2, 1), (3, 2)):
        r = wire.deserialize_response(got[i], params.basis)
        assert np.array_equal(r.ct.raw(), z[f"query_{qi}_ct"])
        assert (r.client_id, r.seq) == tuple(int(v) for v in z[f"query_{qi}_route"])


def test_collector_params_and_unknown_kind(W, params):
    from paper_2604_04696_b200 import server, wire
    col = server.BatchCollector(_DB(8, 8, 32), params)
    out = []
    col.handle_message(wire._frame(wire.KIND_PARAMS, b""), out.append)
    col.handle_message(wire._frame(99, b""), out.append)
    kind, _ = wire.parse_header(out[0])
    assert kind == wire.KIND_PARAMS
    assert server.deserialize_error(out[1]) == (2, "unexpected message kind 99")


# ---------------------------------------------------------------------------
# GPU: the DB container straight to / from HBM, and the collector end to end

@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["pmajor", "transposed"])
def test_gpdb_load_matches_reference(W, params, tag):
    from paper_2604_04696_b200 import wire
    z, m = W
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "db.gpdb")
        open(path, "wb").write(bytes(z[f"gpdb_{tag}"]))
        db, _ = wire.load_database(path, params)
        assert [db.config.d0, db.config.d1, db.config.record_bytes] == m["gpdb_geometry"]
        assert np.array_equal(db.data.astype(np.uint32), z[f"gpdb_{tag}_data"])
        out = os.path.join(td, "out.gpdb")
        wire.save_database(out, db)
        assert open(out, "rb").read() == bytes(z["gpdb_pmajor"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["short", "magic", "truncated"])
def test_gpdb_errors_match_reference(W, params, name):
    from paper_2604_04696_b200 import ParseError, wire
    z, m = W
    msg, off = m["gpdb_bad"][name]
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "bad.gpdb")
        open(path, "wb").write(bytes(z[f"gpdb_bad_{name}"]))
        with pytest.raises(ParseError) as ei:
            wire.load_database(path, params)
    assert str(ei.value) == msg and ei.value.offset == off


@pytest.mark.gpu
def test_collector_end_to_end_bit_exact():
    """Key-set upload + queries as wire bytes through the collector equal
    answer_batch on the same inputs and decrypt to the records."""
    import paper_2604_04696_b200 as G
    from oracle import gpir_oracle as O
    from paper_2604_04696_b200 import server, wire
    from tests.helpers import api_keys, api_query, to_api

    po = O.test_params()
    p = to_api(po)
    d0, d1, rb = 8, 8, 64
    rng = np.random.default_rng(11)
    recs = [rng.integers(0, 256, size=rb, dtype=np.uint8).tobytes() for _ in range(d0 * d1)]
    db = G.encode_database(recs, G.DbConfig(d0, d1, rb), p)
    cli = O.client_keygen(po, d0, d1, rng)
    keys = api_keys(p, cli)
    coords = [(1, 2), (7, 7), (0, 5)]
    qs = [api_query(p, O.client_query(cli, i, j, d0, d1, rng), 5, s) for s, (i, j) in enumerate(coords)]
    want = G.answer_batch(qs, {5: keys}, db, p)
    col = server.BatchCollector(db, p, server.CollectorConfig(batch_max=8, batch_wait_ms=20))
    # upload the key set as the reference client would (evkset message)
    from tests.test_wire import _evkset_bytes
    col.handle_message(_evkset_bytes(5, keys, p), lambda b: None)
    got = {}
    done = threading.Event()
    with col:
        for s, q in enumerate(qs):
            col.handle_message(wire.serialize_query(q), lambda b, s=s: (got.__setitem__(s, b),
                                                                         len(got) == 3 and done.set()))
        assert done.wait(60)
    for s, (i, j) in enumerate(coords):
        r = wire.deserialize_response(got[s], p.basis)
        assert np.array_equal(r.ct.raw(), want[s].ct.raw())
        assert O.decode_plain(O.decrypt(cli, r.ct.raw().astype(np.uint64)), rb, po) == recs[i * d1 + j]


def _evkset_bytes(cid, keys, params):
    """serialize_evkset (src/wire.py:296-302) for the package's ClientKeys."""
    import struct

    from paper_2604_04696_b200 import wire
    g = params.gadget
    parts = [struct.pack("<QHB", cid, len(keys.evks), 1)]
    for e in keys.evks:
        parts.append(struct.pack("<IBH", e.k_aut, g.z_bits, g.ell) + b"".join(wire._ct_body(c) for c in e.ksk))
    parts.append(struct.pack("<BH", g.z_bits, g.ell) + b"".join(wire._ct_body(c) for c in keys.sk_rgsw.rows))
    return wire._frame(wire.KIND_EVKSET, b"".join(parts))
