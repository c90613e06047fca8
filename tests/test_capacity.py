"""Capacity path (GPU): RowSel + the low ColTor stages per power-of-two column
window, batches served as consecutive sub-batches, and compact databases (only
the tensor-core byte-plane image resident, records encoded from device memory).

The tournament pairs columns LSB-first inside every aligned power-of-two window
(/root/reference/pkg/src/latpir/planner.py:457-458, the fact the reference's
column-sharded workers rely on, src/latpir/cluster.py:252-265), and responses do
not depend on batch composition (/root/reference/pkg/tests/test_protocol.py:335-344),
so every forced split must reproduce the oracle's responses bit for bit."""
import numpy as np
import pytest

from oracle import gpir_oracle as O
from tests.helpers import to_api
from tests.test_parity_configs import _answer, _release, _setup

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("window,max_batch", [(32, 0), (64, 16), (0, 7)], ids=["win32", "win64-sub16", "sub7"])
def test_windows_and_subbatches_bitexact(window, max_batch):
    po = O.test_params()
    d0, d1, B = 32, 128, 40  # 2B = 80 > 64: the TMEM-resident RowSel
    G, nat, ctx, h, db, evks, rg, qs, slots = _setup(po, d0, d1, B, seed=window * 7 + max_batch)
    R = po.ring
    try:
        sel = B * window * 2 * R.k * R.n * 4 if window else 0  # the budget that gives this window width
        nat.check(ctx.lib.gpir_set_capacity(ctx.h, sel, max_batch), "capacity")
        out = _answer(nat, ctx, h, qs, slots)
        for _ in range(2):  # graph record + replay of the split pipeline
            assert np.array_equal(_answer(nat, ctx, h, qs, slots), out)
        want = O.answer_batch(qs.astype(np.uint64), evks.astype(np.uint64), rg.astype(np.uint64),
                              db.astype(np.uint64), d0, d1, po)
        assert np.array_equal(out, want)
    finally:
        nat.check(ctx.lib.gpir_set_capacity(ctx.h, 0, 0), "capacity")
        _release(ctx, h, slots)


def test_compact_device_encoded_db():
    import torch

    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200 import _native as nat
    from paper_2604_04696_b200.protocol import get_context

    po = O.test_params()
    p = to_api(po)
    d0, d1, rb, B = 16, 64, 48, 3  # a small batch: compact DBs always take the TMEM-resident RowSel
    rng = np.random.default_rng(55)
    recs = rng.integers(0, 256, size=(d0 * d1, rb), dtype=np.uint8)
    db = G.encode_database_device(torch.from_numpy(recs).cuda(), G.DbConfig(d0, d1, rb), p, compact=True)
    kc = (d0 + 31) // 32 * 32  # K bytes per byte plane, padded to one MMA step
    assert db.device_bytes == d1 * kc * 4 * po.ring.k * po.ring.n  # the byte planes only (d0 = 256: the encoded size)
    with pytest.raises(G.InvalidState):
        _ = db.data
    dbo = O.encode_database([r.tobytes() for r in recs], d0, d1, rb, po)
    total = O.expansion_leaves(d0, d1, po.ell)
    stages = O.expand_stages(total)
    R = po.ring
    uni = lambda *s: np.stack([rng.integers(0, q, size=s + (R.n,), dtype=np.uint32) for q in R.qs], axis=-2)
    evks, rg, qs = uni(B, stages, po.ell, 2), uni(B, 2 * po.ell, 2), uni(B, 2)
    ctx = get_context(p)
    with ctx._lock:
        base = ctx._next
        ctx._next += B
    slots = np.arange(base, base + B, dtype=np.int32)
    try:
        for b in range(B):
            nat.check(ctx.lib.gpir_keys_put(ctx.h, base + b, nat.ptr(np.ascontiguousarray(evks[b])), stages,
                                            nat.ptr(np.ascontiguousarray(rg[b]))), "keys")
        nat.check(ctx.lib.gpir_set_capacity(ctx.h, B * 32 * 2 * R.k * R.n * 4, 2), "capacity")
        out = _answer(nat, ctx, db.handle, qs, slots)
        want = O.answer_batch(qs.astype(np.uint64), evks.astype(np.uint64), rg.astype(np.uint64), dbo, d0, d1, po)
        assert np.array_equal(out, want)
    finally:
        nat.check(ctx.lib.gpir_set_capacity(ctx.h, 0, 0), "capacity")
        with ctx._lock:
            for s in slots:
                ctx.lib.gpir_keys_drop(ctx.h, int(s))
                ctx._free.append(int(s))
