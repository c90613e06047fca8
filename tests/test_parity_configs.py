"""Bit-exact ciphertext parity at the BASELINE configurations (GPU).

Configs 2 (D0=256 x D1=64, B=32) and 3 (256 x 512, B=128) run through the C ABI
(gpir_answer_batch) with the built-in B200 plan -- the plan and kernels the
bench measures: at config 3 the TMEM-resident RowSel (k_rowsel_tk), the A
operand written by the last ExpandQuery stage and the pair-interleaved ColTor
input; at config 2 the M=64 RowSel.  Sampled responses must equal the oracle's
(oracle/gpir_oracle.py, pinned to the live reference) bit for bit.  The oracle
serves each sampled query alone: responses do not depend on batch composition
(batching transparency, /root/reference/pkg/tests/test_protocol.py:335-344).
Key/query/DB material is uniform-random residues (every kernel is
data-oblivious); the DB is uploaded as an NTT-domain P-major tensor
(gpir_db_upload) so the oracle reads the same bytes.

A smaller case on the test ring with B = 40 and 48 (2B > 64: the TMEM-resident
RowSel with a partial second row tile) covers every ColTor executor mode on the
interleaved stage-0 input, against the oracle on the whole batch.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import gpir_oracle as O
from tests.helpers import to_api

pytestmark = pytest.mark.gpu


def _uniform(R, rng, shape):
    return np.stack([rng.integers(0, q, size=shape + (R.n,), dtype=np.uint32) for q in R.qs], axis=-2)


def _setup(po, d0, d1, B, seed):
    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200 import _native as nat
    from paper_2604_04696_b200.protocol import get_context

    R = po.ring
    p = to_api(po)
    rng = np.random.default_rng(seed)
    total = O.expansion_leaves(d0, d1, po.ell)
    stages = O.expand_stages(total)
    db = _uniform(R, rng, (d1, d0)).reshape(d1, d0, R.k * R.n)
    evks = _uniform(R, rng, (B, stages, po.ell, 2))
    rg = _uniform(R, rng, (B, 2 * po.ell, 2))
    qs = _uniform(R, rng, (B, 2))
    ctx = get_context(p)
    h = ctx.lib.gpir_db_upload(ctx.h, nat.ptr(db), d0, d1)
    assert h, nat.last_error()
    with ctx._lock:  # slots outside the ones the package hands out to ClientKeys objects
        base = ctx._next
        ctx._next += B
    for b in range(B):
        nat.check(ctx.lib.gpir_keys_put(ctx.h, base + b, nat.ptr(np.ascontiguousarray(evks[b])), stages,
                                        nat.ptr(np.ascontiguousarray(rg[b]))), "keys")
    slots = np.arange(base, base + B, dtype=np.int32)
    return G, nat, ctx, h, db, evks, rg, qs, slots


def _release(ctx, h, slots):
    with ctx._lock:
        for s in slots:
            ctx.lib.gpir_keys_drop(ctx.h, int(s))
            ctx._free.append(int(s))
    ctx.lib.gpir_db_destroy(ctx.h, h)


def _answer(nat, ctx, h, qs, slots, em=None, cm=None):
    out = np.empty_like(qs)
    e = (nat.ptr(em, C.c_uint8), len(em)) if em is not None else (None, 0)
    c = (nat.ptr(cm, C.c_uint8), len(cm)) if cm is not None else (None, 0)
    nat.check(ctx.lib.gpir_answer_batch(ctx.h, h, nat.ptr(qs), nat.ptr(slots, C.c_int32), len(slots), e[0], e[1],
                                        c[0], c[1], nat.ptr(out), None), "answer")
    return out


@pytest.mark.slow
@pytest.mark.parametrize("d0,d1,B", [(256, 64, 32), (256, 512, 128)], ids=["config2", "config3"])
def test_config_responses_bitexact(d0, d1, B):
    po = O.default_params(plain_bits=16)
    G, nat, ctx, h, db, evks, rg, qs, slots = _setup(po, d0, d1, B, seed=d1 * 7 + B)
    try:
        out = _answer(nat, ctx, h, qs, slots)
        # the graph-replay path (recorded on the second call of the shape, replayed from the third)
        for _ in range(2):
            assert np.array_equal(_answer(nat, ctx, h, qs, slots), out)
        rng = np.random.default_rng(B)
        for b in sorted(set([0, B - 1] + [int(x) for x in rng.choice(B, size=2, replace=False)])):
            want = O.answer_batch(qs[b:b + 1].astype(np.uint64), evks[b:b + 1].astype(np.uint64),
                                  rg[b:b + 1].astype(np.uint64), db, d0, d1, po)
            assert np.array_equal(out[b], want[0]), f"query {b}: response differs from the oracle"
    finally:
        _release(ctx, h, slots)


@pytest.mark.slow
@pytest.mark.parametrize("B", [1, 33], ids=["B1", "B33"])
def test_config3_geometry_other_batches(B):
    """The config-3 DB (256 x 512) at a single query (the streamed-operand RowSel, M = 2)
    and at B = 33 (2B = 66: the TMEM-resident RowSel with a nearly empty row tile), the
    built-in plan: sampled responses equal the oracle's bit for bit."""
    po = O.default_params(plain_bits=16)
    d0, d1 = 256, 512
    G, nat, ctx, h, db, evks, rg, qs, slots = _setup(po, d0, d1, B, seed=300 + B)
    try:
        out = _answer(nat, ctx, h, qs, slots)
        for b in sorted({0, B - 1}):
            want = O.answer_batch(qs[b:b + 1].astype(np.uint64), evks[b:b + 1].astype(np.uint64),
                                  rg[b:b + 1].astype(np.uint64), db, d0, d1, po)
            assert np.array_equal(out[b], want[0]), f"query {b}: response differs from the oracle"
    finally:
        _release(ctx, h, slots)


@pytest.mark.parametrize("B", [40, 48])
@pytest.mark.parametrize("ct_mode", [0, 1, 2, 3], ids=["op", "fused", "split", "hybrid"])
def test_interleaved_coltor_all_modes(B, ct_mode):
    po = O.test_params()
    d0, d1 = 32, 16
    G, nat, ctx, h, db, evks, rg, qs, slots = _setup(po, d0, d1, B, seed=B * 10 + ct_mode)
    try:
        em = np.zeros(16, np.uint8)
        cm = np.full(16, ct_mode, np.uint8)
        out = _answer(nat, ctx, h, qs, slots, em, cm)
        want = O.answer_batch(qs.astype(np.uint64), evks.astype(np.uint64), rg.astype(np.uint64),
                              db.astype(np.uint64), d0, d1, po)
        assert np.array_equal(out, want)
    finally:
        _release(ctx, h, slots)


def test_graphs_with_alternating_batch_classes():
    """Batches alternating between B = 2 (the streamed-operand RowSel, its own DB
    byte-plane layout) and B = 40 (the TMEM-resident RowSel, another layout) with
    CUDA graphs on: each layout change repacks the DB planes and must retire the
    recorded graphs of the other class, so every call stays bit-exact."""
    po = O.test_params()
    d0, d1, B = 32, 64, 40
    G, nat, ctx, h, db, evks, rg, qs, slots = _setup(po, d0, d1, B, seed=4040)
    try:
        nat.check(ctx.lib.gpir_set_graphs(ctx.h, 1), "graphs on")
        want = O.answer_batch(qs.astype(np.uint64), evks.astype(np.uint64), rg.astype(np.uint64),
                              db.astype(np.uint64), d0, d1, po)
        q2, s2 = np.ascontiguousarray(qs[:2]), np.ascontiguousarray(slots[:2])
        for _ in range(4):  # eager, record, replay, replay -- for both classes, interleaved
            assert np.array_equal(_answer(nat, ctx, h, q2, s2), want[:2])
            assert np.array_equal(_answer(nat, ctx, h, qs, slots), want)
    finally:
        _release(ctx, h, slots)
