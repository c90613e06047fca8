"""GPU parity: every kernel and the full server path against the golden
vectors (live reference) and the CPU oracle, bit-exact.  Calls go through the
C ABI (libgpir.so) via the package."""
import numpy as np
import pytest

from oracle import gpir_oracle as O
from tests.helpers import api_keys, api_query, digest, rebuild_case, to_api

pytestmark = pytest.mark.gpu

PROFILES = {
    "tiny": dict(n=64, k=2, prime_bits=20, plain_bits=8, z_bits=7, error_bound=2),
    "proto": dict(),
    "prod": None,
}


def _po(tag):
    return O.default_params() if PROFILES[tag] is None else O.test_params(**PROFILES[tag])


@pytest.fixture(scope="module")
def G():
    import paper_2604_04696_b200 as G
    return G


@pytest.mark.parametrize("tag", list(PROFILES))
def test_ntt_intt_golden(G, golden, tag):
    from paper_2604_04696_b200 import ops
    _, vec = golden
    p = to_api(_po(tag))
    x = vec[f"{tag}_ntt_in"]
    assert np.array_equal(ops.ntt_raw(x, p.basis, p.gadget), vec[f"{tag}_ntt_out"])
    assert np.array_equal(ops.intt_raw(x, p.basis, p.gadget), vec[f"{tag}_intt_out"])


@pytest.mark.parametrize("tag", list(PROFILES))
def test_ntt_roundtrip_many(G, tag):
    from paper_2604_04696_b200 import ops
    po = _po(tag)
    p = to_api(po)
    rng = np.random.default_rng(7)
    x = np.stack([rng.integers(0, q, size=(300, po.n), dtype=np.uint64) for q in po.ring.qs], axis=1)
    f = ops.ntt_raw(x, p.basis, p.gadget)
    assert np.array_equal(f, O.ntt(x, po.ring))
    assert np.array_equal(ops.intt_raw(f, p.basis, p.gadget), x)
    # edge values: zeros and q-1 everywhere
    e = np.zeros_like(x[:2])
    e[1] = po.ring.q - 1
    assert np.array_equal(ops.ntt_raw(e, p.basis, p.gadget), O.ntt(e, po.ring))


@pytest.mark.parametrize("tag", list(PROFILES))
def test_digits_golden(G, golden, tag):
    from paper_2604_04696_b200 import ops
    _, vec = golden
    p = to_api(_po(tag))
    d = ops.digits(vec[f"{tag}_ntt_in"], p.basis, p.gadget)
    assert np.array_equal(d, vec[f"{tag}_digits"])


@pytest.mark.parametrize("tag", list(PROFILES))
def test_digits_extremes(G, tag):
    from paper_2604_04696_b200 import ops
    po = _po(tag)
    p = to_api(po)
    R = po.ring
    # coefficients 0, +-1, +-(Q-1)/2 and around z/2 boundaries, written as residues
    vals = [0, 1, -1, (R.Q - 1) // 2, -((R.Q - 1) // 2), (1 << (po.z_bits - 1)), (1 << (po.z_bits - 1)) + 1,
            -(1 << (po.z_bits - 1)) - 1, (1 << (2 * po.z_bits - 1)) + (1 << (po.z_bits - 1)) + 1]
    x = np.zeros((1, R.k, R.n), dtype=np.uint64)
    for j, v in enumerate(vals):
        for i, q in enumerate(R.qs):
            x[0, i, j] = v % q
    assert np.array_equal(ops.digits(x, p.basis, p.gadget), O.gadget_digits(x, R, po.z_bits, po.ell))


@pytest.mark.parametrize("tag", list(PROFILES))
@pytest.mark.parametrize("mode", ["op", "stage", "split", "hybrid"])
def test_subs_and_external_product_golden(G, golden, tag, mode):
    from paper_2604_04696_b200 import ops
    _, vec = golden
    po = _po(tag)
    p = to_api(po)
    m = mode
    st, ks = vec[f"{tag}_subs_in"], vec[f"{tag}_subs_ksk"]
    out = ops.expand_stage(st, ks, po.n // 2 + 1, None, p.basis, p.gadget, m)
    assert np.array_equal(out, vec[f"{tag}_subs_out"])
    xp = ops.external_product_batch(st, vec[f"{tag}_xp_rows"], p.basis, p.gadget, m)
    assert np.array_equal(xp, vec[f"{tag}_xp_out"])


@pytest.mark.parametrize("mode", ["op", "stage", "split", "hybrid"])
def test_expand_stages_and_coltor_vs_oracle(G, mode):
    from paper_2604_04696_b200 import ops
    po = O.default_params()
    p = to_api(po)
    R = po.ring
    m = mode
    rng = np.random.default_rng(99)
    uni = lambda *s: np.stack([rng.integers(0, q, size=s + (R.n,), dtype=np.uint64) for q in R.qs], axis=-2)
    B, C = 3, 4
    st = uni(B, C, 2)
    ks = uni(B, po.ell, 2)
    for t in (0, 3, 8, 11):
        got = ops.expand_stage(st, ks, R.n // (1 << t) + 1, None, p.basis, p.gadget, m)
        assert np.array_equal(got, O.subs_stage(st, ks, R.n // (1 << t) + 1, t, po)), t
    rows = uni(B, 2 * po.ell, 2)
    got = ops.coltor_stage(st, rows, p.basis, p.gadget, m)
    even, odd = st[:, 0::2], st[:, 1::2]
    want = (even + O.ext_product((odd + R.q - even) % R.q, rows, po)) % R.q
    assert np.array_equal(got, want)


@pytest.mark.parametrize("tag", list(PROFILES))
def test_rowsel_golden(G, golden, tag):
    from types import SimpleNamespace

    from paper_2604_04696_b200 import ops
    _, vec = golden
    po = _po(tag)
    p = to_api(po)
    R = po.ring
    a = vec[f"{tag}_gemm_a"].astype(np.uint64)
    d = vec[f"{tag}_gemm_b"].astype(np.uint64)
    rows = a.reshape(2, 2, 5, R.k, R.n).transpose(0, 2, 1, 3, 4)
    fake = SimpleNamespace(config=G.DbConfig(5, 2, 1), params=p, data=d, layout=G.LayoutKind.P_MAJOR)
    sel = ops.row_select(rows, fake, p)
    want = vec[f"{tag}_gemm_out"].reshape(2, 2, 2, R.k, R.n).transpose(0, 2, 1, 3, 4)
    assert np.array_equal(sel, want)


@pytest.mark.parametrize("engine", ["cudacore", "tensorcore"])
@pytest.mark.parametrize("shape", [(1, 5, 2), (3, 64, 16), (32, 70, 64), (64, 256, 128), (17, 129, 1), (65, 64, 32), (128, 130, 64)])
def test_rowsel_engines_vs_oracle(G, engine, shape):
    """Both RowSel engines, ragged shapes (B, d0, d1) incl. M = 2B = 128 and > 128 (row tiles), d0 not a
    multiple of the 64-byte K chunk, d1 below and above the 32-column tile,
    and residues at q-1 (largest byte planes)."""
    from types import SimpleNamespace

    from paper_2604_04696_b200 import ops
    B, d0, d1 = shape
    po = O.test_params()
    p = to_api(po)
    R = po.ring
    rng = np.random.default_rng(B * 1000 + d0 + d1)
    rows = np.stack([rng.integers(0, q, size=(B, d0, 2, R.n), dtype=np.uint64) for q in R.qs], axis=-2)
    db = np.stack([rng.integers(0, q, size=(d1, d0, R.n), dtype=np.uint64) for q in R.qs], axis=-2)
    rows[0, 0] = R.q - 1
    db[0, :] = R.q - 1
    db = db.reshape(d1, d0, R.k * R.n)
    fake = SimpleNamespace(config=G.DbConfig(d0, d1, 1), params=p, data=db, layout=G.LayoutKind.P_MAJOR)
    assert np.array_equal(ops.row_select(rows, fake, p, engine=engine), O.rowsel(rows, db, R))


@pytest.mark.parametrize("engine", ["pmajor", "tensorcore"])
def test_pipeline_rowsel_engines(G, golden, engine):
    cases, _ = golden
    case = cases["prod_16x16"]
    po, records, clients, queries = rebuild_case(case)
    p = to_api(po)
    db = G.encode_database(records, G.DbConfig(16, 16, case["record_bytes"]), p)
    keys = {cid: api_keys(p, c) for cid, c in clients.items()}
    qs = [api_query(p, q, cid) for q, (cid, _, _) in zip(queries, case["queries"])]
    out = np.stack([r.ct.raw() for r in G.answer_batch(qs, keys, db, p, engine=engine)])
    assert digest(out) == case["digest"]["responses"]


def test_rowsel_large_k_fold(G):
    """D0 > 1024 exercises the periodic mod-q fold (src/layout.py:185-187)."""
    from types import SimpleNamespace

    from paper_2604_04696_b200 import ops
    po = O.test_params()
    p = to_api(po)
    R = po.ring
    rng = np.random.default_rng(5)
    d0, d1, B = 1100, 3 * 0 + 2, 2
    rows = np.stack([rng.integers(q - 1000, q, size=(B, d0, 2, R.n), dtype=np.uint64) for q in R.qs], axis=-2)
    db = np.stack([rng.integers(q - 1000, q, size=(d1, d0, R.n), dtype=np.uint64) for q in R.qs], axis=-2)
    db = db.reshape(d1, d0, R.k * R.n)
    fake = SimpleNamespace(config=G.DbConfig(d0, d1, 1), params=p, data=db, layout=G.LayoutKind.P_MAJOR)
    assert np.array_equal(ops.row_select(rows, fake, p), O.rowsel(rows, db, R))


def _run_case(G, case, mode=None, plan=None, split=False):
    po, records, clients, queries = rebuild_case(case)
    p = to_api(po)
    cfg = G.DbConfig(case["d0"], case["d1"], case["record_bytes"])
    db = G.encode_database(records, cfg, p)
    keys = {cid: api_keys(p, c) for cid, c in clients.items()}
    qs = [api_query(p, q, cid, s) for s, (q, (cid, _, _)) in enumerate(zip(queries, case["queries"]))]
    if split:
        resp = [G.respond(q, keys[q.client_id], db, p, mode=mode) for q in qs]
    else:
        resp = G.answer_batch(qs, keys, db, p, mode=mode, plan=plan)
    return po, records, clients, db, np.stack([r.ct.raw() for r in resp]), resp


@pytest.mark.parametrize("name", ["proto_8x8", "proto_5x1", "prod_4x4", "prod_16x16", "prod_p16_256x2"])
def test_pipeline_golden(G, golden, name):
    cases, vec = golden
    case = cases[name]
    po, records, clients, db, out, resp = _run_case(G, case)
    assert digest(db.data) == case["digest"]["db"], "GPU DB encode differs from the reference"
    assert digest(out) == case["digest"]["responses"], "GPU responses differ from the reference"
    if f"{name}_responses" in vec.files:
        assert np.array_equal(out, vec[f"{name}_responses"])
    if f"{name}_responses_head" in vec.files:
        assert np.array_equal(out[..., :64], vec[f"{name}_responses_head"])
    for (cid, i, j), ct, r in zip(case["queries"], out, resp):
        assert r.client_id == cid
        assert O.decode_plain(O.decrypt(clients[cid], ct), case["record_bytes"], po) == records[i * case["d1"] + j]


@pytest.mark.parametrize("mode", ["op", "stage"])
def test_execution_modes_and_batching_transparency(G, golden, mode):
    cases, _ = golden
    case = cases["prod_4x4"]
    m = G.ExecMode.STAGE_LEVEL if mode == "stage" else G.ExecMode.OPERATION_LEVEL
    *_, out_b, _ = _run_case(G, case, mode=m)
    *_, out_s, _ = _run_case(G, case, mode=m, split=True)
    assert digest(out_b) == case["digest"]["responses"]
    assert np.array_equal(out_b, out_s)


def test_errors(G, golden):
    cases, _ = golden
    case = cases["proto_8x8"]
    po, records, clients, queries = rebuild_case(case)
    p = to_api(po)
    db = G.encode_database(records, G.DbConfig(8, 8, 64), p)
    q = api_query(p, queries[0], 5)
    with pytest.raises(G.InvalidState):
        G.answer_batch([q], {}, db, p)
    with pytest.raises(G.InvalidArgument):
        G.answer_batch([q], {5: api_keys(p, clients[0])}, db, p, engine="bogus")
    assert G.answer_batch([], {}, db, p) == []
    with pytest.raises(G.InvalidArgument):
        G.encode_database(records[:-1], G.DbConfig(8, 8, 64), p)
    with pytest.raises(G.InvalidArgument):
        G.encode_database([b"x" * 65] + records[1:], G.DbConfig(8, 8, 64), p)


def test_reference_encoded_db_upload_roundtrip(G, golden):
    """A P-major tensor from the oracle/reference uploads into the brv layout and back."""
    from types import SimpleNamespace
    cases, _ = golden
    case = cases["prod_4x4"]
    po, records, clients, queries = rebuild_case(case)
    p = to_api(po)
    data = O.encode_database(records, 4, 4, case["record_bytes"], po)
    ref_db = SimpleNamespace(config=G.DbConfig(4, 4, case["record_bytes"]), params=p, data=data,
                             layout=G.LayoutKind.P_MAJOR)
    up = G.upload_database(ref_db)
    assert np.array_equal(up.data, data)
    keys = {7: api_keys(p, clients[7])}
    qs = [api_query(p, q, 7) for q in queries]
    out = np.stack([r.ct.raw() for r in G.answer_batch(qs, keys, ref_db, p)])
    assert digest(out) == case["digest"]["responses"]


def test_full_size_decrypt_property(G):
    """Config-2 geometry (D0=256, D1=64, P=2^16, 8 KiB records) with 3 distinct
    clients: every decrypted response equals the DB record (size-independent
    property at the full size; the oracle would take minutes here)."""
    po = O.default_params(plain_bits=16)
    p = to_api(po)
    d0, d1, rb = 256, 64, 8192
    rng = np.random.default_rng(20261017)
    buf = rng.integers(0, 256, size=(d0 * d1, rb), dtype=np.uint8)
    db = G.encode_database_array(buf, G.DbConfig(d0, d1, rb), p)
    clients = {c: O.client_keygen(po, d0, d1, rng) for c in (11, 12, 13)}
    keys = {c: api_keys(p, cl) for c, cl in clients.items()}
    targets = [(11, 0, 0), (12, 255, 63), (13, 128, 17), (11, 3, 62)]
    qs = [api_query(p, O.client_query(clients[c], i, j, d0, d1, rng), c, s) for s, (c, i, j) in enumerate(targets)]
    resp = G.answer_batch(qs, keys, db, p)
    for (c, i, j), r in zip(targets, resp):
        m = O.decrypt(clients[c], r.ct.raw())
        assert O.decode_plain(m, rb, po) == buf[i * d1 + j].tobytes()


@pytest.mark.parametrize("name", ["prod_4x4", "proto_8x8"])
def test_graph_replay_matches_eager(G, golden, name):
    """Calls without per-phase stats record the pipeline as a CUDA graph on the
    second call of a shape and replay it from the third: with new query contents
    every replay must equal the eager path (stats requested), and the first
    batch must still decrypt to its records."""
    from paper_2604_04696_b200 import protocol
    cases, _ = golden
    case = cases[name]
    po, records, clients, db, out0, resp = _run_case(G, case)
    p = to_api(po)
    keys = {cid: api_keys(p, c) for cid, c in clients.items()}
    ids = [cid for cid, _, _ in case["queries"]]
    q0 = np.stack([r.ct.raw() for r in resp])  # any valid (B, 2, k, n) input shape; contents vary below
    qs = [api_query(p, q, cid, s) for s, (q, (cid, _, _)) in
          enumerate(zip(rebuild_case(case)[3], case["queries"]))]
    first = np.stack([q.ct.raw() for q in qs]).astype(np.uint32)
    rng = np.random.default_rng(17)
    qmod = np.array(po.ring.qs, dtype=np.uint64)[:, None]
    batches = [first] + [(rng.integers(0, 1 << 62, size=q0.shape, dtype=np.uint64) % qmod).astype(np.uint32)
                         for _ in range(4)] + [first]
    for i, qa in enumerate(batches):
        g = protocol.answer_raw(np.ascontiguousarray(qa), ids, keys, db, p)          # graph path (3rd call on)
        e = protocol.answer_raw(np.ascontiguousarray(qa), ids, keys, db, p, stats=G.ServeStats())  # eager
        assert np.array_equal(g, e), f"batch {i}: graph replay differs from the eager pipeline"
        if i in (0, len(batches) - 1):
            assert np.array_equal(g, out0)


def test_caller_graph_capture(G, golden):
    """A caller may record gpir_answer_batch_dev into its own CUDA graph (torch.cuda.CUDAGraph):
    the library then launches eagerly into the caller's capture; replays equal the eager result."""
    import ctypes as C

    import torch

    from paper_2604_04696_b200 import _native as nat
    from paper_2604_04696_b200 import protocol
    cases, _ = golden
    case = cases["prod_4x4"]
    po, records, clients, db, out0, resp = _run_case(G, case)
    p = to_api(po)
    keys = {cid: api_keys(p, c) for cid, c in clients.items()}
    ids = [cid for cid, _, _ in case["queries"]]
    qs = [api_query(p, q, cid, s) for s, (q, (cid, _, _)) in
          enumerate(zip(rebuild_case(case)[3], case["queries"]))]
    qarr = np.stack([q.ct.raw() for q in qs]).astype(np.uint32)
    protocol.answer_raw(qarr, ids, keys, db, p)  # keys into their slots
    ddb = protocol._device_db(db, p)
    ctx = ddb.ctx
    stages = G.planner.num_expand_stages(G.planner.expansion_leaves(db.config.d0, db.config.d1, p.gadget.ell))
    slots = torch.tensor([ctx.key_slot(keys[c], stages, db.config.d1 > 1) for c in ids], dtype=torch.int32).pin_memory()
    d_q = torch.from_numpy(qarr.view(np.int32)).cuda()
    d_o = torch.empty_like(d_q)
    em = np.zeros(16, np.uint8)
    cm = np.zeros(16, np.uint8)
    nat.check(ctx.lib.gpir_plan(ctx.h, db.config.d0, db.config.d1, len(ids), nat.ptr(em, C.c_uint8), 16,
                                nat.ptr(cm, C.c_uint8), 16), "plan")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        def call():
            nat.check(ctx.lib.gpir_answer_batch_dev(ctx.h, ddb.handle, C.c_void_p(d_q.data_ptr()),
                                                    C.cast(C.c_void_p(slots.data_ptr()), C.POINTER(C.c_int32)),
                                                    len(ids), nat.ptr(em, C.c_uint8), 16, nat.ptr(cm, C.c_uint8), 16,
                                                    C.c_void_p(d_o.data_ptr()), C.c_void_p(s.cuda_stream), None),
                      "answer_dev")
        call()  # eager once (lazy allocations)
        s.synchronize()
        g.capture_begin()
        call()
        g.capture_end()
    for _ in range(2):
        d_o.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(d_o.cpu().numpy().view(np.uint32).reshape(out0.shape), out0)


def test_digits_boundary_vectors(G):
    """The production-ring (z = 2^22) closed-form digit kernel against the reference's own
    DigitExtractor on crafted boundary coefficients (tests/golden/digits_boundary.npz,
    tools/make_digit_golden.py): raw digit == z/2 stays positive, z/2 + 1 carries, carry
    chains through all ell digits, +-(Q-1)/2."""
    import os

    from paper_2604_04696_b200 import ops
    v = np.load(os.path.join(os.path.dirname(__file__), "golden", "digits_boundary.npz"))
    p = to_api(O.default_params())
    got = ops.digits(v["coeff"].astype(np.uint64), p.basis, p.gadget)
    assert np.array_equal(got, v["digits"].astype(np.int64))
