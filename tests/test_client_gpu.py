"""GPU client factory (paper_2604_04696_b200.client): keys installed straight
into key slots and queries encrypted on the GPU must be served correctly --
every response decrypts (with the oracle's decryption) to the selected record."""
import numpy as np
import pytest

from oracle import gpir_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d0,d1,rb,pb", [(16, 8, 1024, 16), (8, 1, 2048, 16), (32, 4, 8192, 16)])
def test_gpu_clients_decrypt(d0, d1, rb, pb):
    import ctypes as C

    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200 import _native as nat
    from paper_2604_04696_b200 import client
    from tests.helpers import to_api

    po = O.default_params(plain_bits=pb)
    p = to_api(po)
    R = po.ring
    rng = np.random.default_rng(d0 * 100 + d1)
    recs = rng.integers(0, 256, size=(d0 * d1, rb), dtype=np.uint8)
    db = G.encode_database_array(recs, G.DbConfig(d0, d1, rb), p)
    ctx = db.ctx
    B = 4
    secrets = [client.keygen(ctx, p, 40 + b, d0, d1, seed=1000 + b) for b in range(B)]
    coords = [(int(rng.integers(0, d0)), int(rng.integers(0, d1))) for _ in range(B)]
    qs = np.concatenate([client.queries(ctx, p, secrets[b], d0, d1, [coords[b]], seed=77 + b) for b in range(B)])
    slots = np.arange(40, 40 + B, dtype=np.int32)
    out = np.empty_like(qs)
    nat.check(ctx.lib.gpir_answer_batch(ctx.h, db.handle, nat.ptr(qs), nat.ptr(slots, C.c_int32), B, None, 0, None, 0,
                                        nat.ptr(out), None), "answer")
    for b in range(B):
        assert set(np.unique(secrets[b])) <= {-1, 0, 1}
        s = O.ntt((secrets[b].astype(np.int64)[None] % R.q_i64).astype(np.uint64), R)
        cli = O.Client(po, s, None, None)
        i, j = coords[b]
        got = O.decode_plain(O.decrypt(cli, out[b].astype(np.uint64)), rb, po)
        assert got == recs[i * d1 + j].tobytes(), (b, i, j)


@pytest.mark.parametrize("d0,d1,B", [(256, 64, 32), (256, 512, 128)])
def test_full_size_configs_decrypt(d0, d1, B):
    """BASELINE configs 2 and 3 at full size (1 GiB / 8 GiB encoded DB, B distinct
    GPU-generated clients, the built-in B200 plan): every sampled response
    decrypts to its record (a size-independent correctness property)."""
    import ctypes as C

    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200 import _native as nat
    from paper_2604_04696_b200 import client
    from tests.helpers import to_api

    rb = 8192
    po = O.default_params(plain_bits=16)
    p = to_api(po)
    R = po.ring
    rng = np.random.default_rng(d1)
    recs = rng.integers(0, 256, size=(d0 * d1, rb), dtype=np.uint8)
    db = G.encode_database_array(recs, G.DbConfig(d0, d1, rb), p)
    ctx = db.ctx
    coords = [(int(rng.integers(0, d0)), int(rng.integers(0, d1))) for _ in range(B)]
    secrets = [client.keygen(ctx, p, b, d0, d1, seed=31 * b + 1) for b in range(B)]
    qs = np.concatenate([client.queries(ctx, p, secrets[b], d0, d1, [coords[b]], seed=17 * b + 3) for b in range(B)])
    out = np.empty_like(qs)
    slots = np.arange(B, dtype=np.int32)
    nat.check(ctx.lib.gpir_answer_batch(ctx.h, db.handle, nat.ptr(qs), nat.ptr(slots, C.c_int32), B, None, 0, None, 0,
                                        nat.ptr(out), None), "answer")
    for b in rng.choice(B, size=4, replace=False):
        s = O.ntt((secrets[b].astype(np.int64)[None] % R.q_i64).astype(np.uint64), R)
        i, j = coords[b]
        got = O.decode_plain(O.decrypt(O.Client(po, s, None, None), out[b].astype(np.uint64)), rb, po)
        assert got == recs[i * d1 + j].tobytes(), (b, i, j)
