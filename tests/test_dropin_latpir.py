"""Drop-in with the reference's own objects (GPU): latpir's HeParams, ClientKeys,
ClientQuery and EncodedDatabase go straight into paper_2604_04696_b200.answer_batch
/ respond, the responses come back as latpir Response objects, equal the ones
latpir.protocol.answer_batch computes on the CPU bit for bit, and latpir's
ClientSession.decode recovers the records (/root/reference/pkg/src/latpir/
protocol.py:605-688).  latpir is the unmodified reference installed in
baseline/_ref (git-ignored; it travels to the GPU box with the repo snapshot);
the test skips when it is absent.  Also: tile / pipeline configurations the
reference rejects raise the same InvalidConfig here, and ServeStats.stages gets
one entry per stage."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not os.path.isdir(os.path.join(REF, "latpir")):
        pytest.skip("latpir (the reference) is not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import latpir.he
    import latpir.layout
    import latpir.protocol
    return latpir


def _world(L, P, d0, d1, rb, seed):
    LP = L.protocol
    cfg = LP.DbConfig(d0, d1, rb)
    rng = np.random.default_rng(seed)
    recs = [rng.integers(0, 256, size=rb, dtype=np.uint8).tobytes() for _ in range(cfg.records)]
    db = LP.encode_database(recs, cfg, P)
    sess = [LP.ClientSession.create(P, cfg, rng, client_id=c) for c in (3, 7)]
    return cfg, recs, db, sess, rng


@pytest.mark.parametrize("profile", ["test", "production"])
def test_reference_objects_through_answer_batch(L, profile):
    import paper_2604_04696_b200 as G

    LP = L.protocol
    if profile == "test":
        P, (d0, d1, rb) = L.he.test_params(), (8, 8, 32)
    else:
        P, (d0, d1, rb) = L.he.default_params(), (4, 4, 1024)
    cfg, recs, db, sess, rng = _world(L, P, d0, d1, rb, seed=11)
    keys = {s.client_id: s.keys for s in sess}
    targets = [(1, 2), (d0 - 1, d1 - 1), (0, 3)]
    qs = [sess[i % 2].gen_query(a, b, rng) for i, (a, b) in enumerate(targets)]
    ours = G.answer_batch(qs, keys, db, P)
    theirs = LP.answer_batch(qs, keys, db, P)
    for o, t, q, (a, b) in zip(ours, theirs, qs, targets):
        assert type(o) is type(t)
        assert (o.client_id, o.seq) == (t.client_id, t.seq)
        assert np.array_equal(o.ct.a.limbs, t.ct.a.limbs) and np.array_equal(o.ct.b.limbs, t.ct.b.limbs)
        s = next(x for x in sess if x.client_id == q.client_id)
        assert s.decode(o) == recs[a * cfg.d1 + b]
    one = G.respond(qs[0], keys[qs[0].client_id], db, P)
    assert np.array_equal(one.ct.a.limbs, theirs[0].ct.a.limbs)


def test_tile_pipeline_validation_matches_reference(L):
    import paper_2604_04696_b200 as G

    P = L.he.test_params()
    cfg, recs, db, sess, rng = _world(L, P, 8, 8, 32, seed=12)
    keys = {s.client_id: s.keys for s in sess}
    qs = [sess[0].gen_query(1, 1, rng)]
    TC, PC = L.layout.TileConfig, L.layout.PipelineConfig
    bad = [dict(tile=TC(3, 8, 8, bp=1)), dict(tile=TC(2, 8, 8)),  # bm does not divide 2B; p-major needs bp
           dict(pipeline=PC(prime_streams=3)), dict(pipeline=PC(n_chunks=7))]
    for kw in bad:
        with pytest.raises(L.errors.InvalidConfig if hasattr(L, "errors") else Exception):
            L.protocol.answer_batch(qs, keys, db, P, **kw)
        with pytest.raises(G.InvalidConfig):
            G.answer_batch(qs, keys, db, P, **kw)
    good = dict(tile=TC(2, 8, 8, bp=4), pipeline=None)
    out = G.answer_batch(qs, keys, db, P, **good)
    assert np.array_equal(out[0].ct.a.limbs, L.protocol.answer_batch(qs, keys, db, P, **good)[0].ct.a.limbs)


def test_serve_stats_stages(L):
    import paper_2604_04696_b200 as G

    P = L.he.test_params()
    cfg, recs, db, sess, rng = _world(L, P, 8, 8, 32, seed=13)
    keys = {s.client_id: s.keys for s in sess}
    qs = [sess[0].gen_query(1, 1, rng), sess[1].gen_query(2, 3, rng)]
    st = G.ServeStats()
    G.answer_batch(qs, keys, db, P, stats=st)
    phases = [s.phase for s in st.stages]
    n_eq = G.planner.num_expand_stages(G.planner.expansion_leaves(8, 8, P.gadget.ell))
    assert phases.count("ExpandQuery") == n_eq and phases.count("ColTor") == 3
    assert "RowSel" in phases and "RgswAssembly" in phases
    assert all(s.seconds > 0 for s in st.stages)
    assert set(st.phase_seconds) >= {"ExpandQuery", "RgswAssembly", "RowSel", "ColTor"}
