"""Row-sharded multi-rank serving (paper_2604_04696_b200.cluster).

CPU: world_size-2 gloo processes run the real orchestration and NCCL-style
collectives with the oracle as the per-rank compute backend; the combined
responses must equal the single-process pipeline bit for bit.
GPU: two virtual ranks on one device (threads + an in-process transport)
drive the real C-ABI sharded kernels; responses must equal the oracle's."""
import os
import threading

import numpy as np
import pytest
import torch

from oracle import gpir_oracle as O

D0, D1, RB = 8, 4, 32


class OracleRowShard:
    """Oracle compute for one rank (tests only)."""

    def __init__(self, po, db_pm_local, d0, d1, clients_own):
        self.po, self.db, self.d0, self.d1 = po, db_pm_local, d0, d1
        self.clients = clients_own
        R = po.ring
        self.ct = 2 * R.k * R.n

    def swap01(self, x):
        return x.transpose(0, 1).contiguous()

    def expand(self, q_own, _slots):
        R = self.po.ring
        qs = q_own.numpy().astype(np.uint64).reshape(-1, 2, R.k, R.n)
        evks = np.stack([c.evks for c in self.clients])
        leaves = O.expand(qs, evks, self.d0, self.d1, self.po)
        self.leaves = leaves
        return torch.from_numpy(leaves[:, :self.d0].reshape(len(qs), self.d0, self.ct).astype(np.int64))

    def rowsel(self, rows_all):
        R = self.po.ring
        rows = rows_all.numpy().astype(np.uint64).reshape(rows_all.shape[0], -1, 2, R.k, R.n)
        sel = O.rowsel(rows, self.db, R)
        return torch.from_numpy(sel.reshape(sel.shape[0], self.d1, self.ct).astype(np.int64))

    def coltor(self, sums):
        R = self.po.ring
        sel = sums.numpy().astype(np.uint64).reshape(sums.shape[0], self.d1, 2, R.k, R.n) % R.q
        rg = O.build_rgsw(self.leaves[:, self.d0:], np.stack([c.sk_rgsw for c in self.clients]), self.po)
        out = O.coltor(sel, rg, self.po)
        return torch.from_numpy(out.reshape(out.shape[0], self.ct).astype(np.int64))


def _material(po, n_queries, seed=3):
    rng = np.random.default_rng(seed)
    recs = [rng.integers(0, 256, size=RB, dtype=np.uint8).tobytes() for _ in range(D0 * D1)]
    clients = [O.client_keygen(po, D0, D1, rng) for _ in range(n_queries)]
    targets = [(int(rng.integers(0, D0)), int(rng.integers(0, D1))) for _ in range(n_queries)]
    qs = [O.client_query(c, i, j, D0, D1, rng) for c, (i, j) in zip(clients, targets)]
    return recs, clients, targets, np.stack(qs)


def _rank_main(rank, world, port, out_path):
    import torch.distributed as dist

    from paper_2604_04696_b200.cluster import CountingComm, TorchComm, answer_row_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    po = O.test_params()
    B = 2 * world
    recs, clients, _, qs = _material(po, B)
    db = O.encode_database(recs, D0, D1, RB, po)               # (d1, d0, kn)
    d0l = D0 // world
    db_local = np.ascontiguousarray(db[:, rank * d0l:(rank + 1) * d0l])
    own = slice(rank * B // world, (rank + 1) * B // world)
    be = OracleRowShard(po, db_local, D0, D1, clients[own])
    q_own = torch.from_numpy(qs[own].astype(np.int64))
    cc = CountingComm(TorchComm())
    out = answer_row_sharded(be, cc, q_own, None, D0, D1)
    np.save(out_path + f".{rank}.npy", out.numpy())
    np.save(out_path + f".ledger.{rank}.npy", np.array([cc.ledger.after_expand_bytes, cc.ledger.after_coltor_bytes,
                                                         cc.ledger.rgsw_sidecar_bytes], dtype=np.int64))
    dist.barrier()
    dist.destroy_process_group()


def test_row_sharded_gloo_matches_single_process(tmp_path):
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    path = str(tmp_path / "resp")
    mp.start_processes(_rank_main, args=(world, port, path), nprocs=world, start_method="spawn", join=True)
    got = np.concatenate([np.load(path + f".{r}.npy") for r in range(world)]).astype(np.uint64)
    po = O.test_params()
    B = 2 * world
    _check_ledger(path, world, "row", po, B)
    recs, clients, targets, qs = _material(po, B)
    db = O.encode_database(recs, D0, D1, RB, po)
    want = O.answer_batch(qs, np.stack([c.evks for c in clients]), np.stack([c.sk_rgsw for c in clients]), db,
                          D0, D1, po)
    R = po.ring
    assert np.array_equal(got.reshape(want.shape), want)
    for c, (i, j), ct in zip(clients, targets, want):
        assert O.decode_plain(O.decrypt(c, ct), RB, po) == recs[i * D1 + j]


def _check_ledger(path, world, mode, po, B):
    """The bytes the run's collectives moved (CountingComm, summed over ranks) equal the
    closed-form device ledger (cluster.device_comm_bytes; reference: comm_bytes,
    src/cluster.py:124-136).  The oracle backend moves int64 words: 2x the u32 volume."""
    from paper_2604_04696_b200.cluster import Strategy, device_comm_bytes
    from paper_2604_04696_b200.values import DbConfig
    from tests.helpers import to_api

    got = sum(np.load(path + f".ledger.{r}.npy") for r in range(world))
    st = Strategy.ROW_SHARD if mode == "row" else Strategy.SHARD_ALL_GATHER
    led = device_comm_bytes(st, DbConfig(D0, D1, RB), B, world, to_api(po))
    assert list(got) == [2 * led.after_expand_bytes, 2 * led.after_coltor_bytes, 2 * led.rgsw_sidecar_bytes]


def test_bench_spawns_ranks_cpu():
    """`bench.py --gpus 2` re-launches itself under torchrun (2 ranks, 127.0.0.1);
    the reference arm runs on rank 0 alone and prints one JSON line with n_gpus 2."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "1", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference" and d["value"] > 0
    assert d["config"]["parallelism"].startswith("replica2")  # B = 1 does not split over 2 ranks


def test_comm_ledger_closed_forms():
    """Reference-format ledger (wire bytes, src/cluster.py:124-136) and the device volumes of
    both sharded modes at config 4 on 8 GPUs."""
    from paper_2604_04696_b200 import default_params, wire
    from paper_2604_04696_b200.cluster import Strategy, comm_bytes, device_comm_bytes
    from paper_2604_04696_b200.values import DbConfig

    p = default_params()
    cfg = DbConfig(256, 2048, 8192)
    ct = wire.serialized_ct_bytes(p)
    led = comm_bytes(Strategy.SHARD_ALL_GATHER, cfg, 256, 8, p)
    assert led.after_expand_bytes == 256 * 256 * ct and led.after_coltor_bytes == 256 * 8 * ct
    assert comm_bytes(Strategy.NAIVE_BATCH, cfg, 256, 8, p).after_expand_bytes == 0
    row = device_comm_bytes(Strategy.ROW_SHARD, cfg, 256, 8, p)
    assert row.after_coltor_bytes == 7 * 256 * 2048 * 131072  # 56 GiB per rank: grows with the DB
    col = device_comm_bytes(Strategy.SHARD_ALL_GATHER, cfg, 256, 8, p)
    assert col.after_expand_bytes == 7 * 256 * 256 * 131072 and col.after_coltor_bytes == 7 * 256 * 131072


class _ThreadComm:
    """In-process transport for n threads (one per virtual rank)."""

    def __init__(self, n):
        self.n = n
        self.bar = threading.Barrier(n)
        self.slots = [None] * n

    def view(self, rank):
        outer = self

        class V:
            size = outer.n

            def all_to_all(self, send):
                outer.slots[rank] = send
                outer.bar.wait()
                recv = torch.stack([outer.slots[s][rank] for s in range(outer.n)])
                outer.bar.wait()
                return recv

            def reduce_scatter_sum(self, x):
                outer.slots[rank] = x
                outer.bar.wait()
                out = sum(outer.slots[s][rank] for s in range(outer.n))
                outer.bar.wait()
                return out

            def all_gather(self, x):
                outer.slots[rank] = x
                outer.bar.wait()
                out = torch.stack([outer.slots[s] for s in range(outer.n)])
                outer.bar.wait()
                return out

        return V()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 4])
def test_row_sharded_gpu_virtual_ranks(world):
    from paper_2604_04696_b200.cluster import CudaRowShard, answer_row_sharded
    from tests.helpers import to_api

    po = O.default_params(plain_bits=16)
    p = to_api(po)
    d0, d1, rb = 16, 8, 1024
    B = 2 * world
    rng = np.random.default_rng(77)
    recs = rng.integers(0, 256, size=(d0 * d1, rb), dtype=np.uint8)
    clients = [O.client_keygen(po, d0, d1, rng) for _ in range(B)]
    targets = [(int(rng.integers(0, d0)), int(rng.integers(0, d1))) for _ in range(B)]
    qs = np.stack([O.client_query(c, i, j, d0, d1, rng) for c, (i, j) in zip(clients, targets)])
    comm = _ThreadComm(world)
    d0l = d0 // world
    bes, outs = [], [None] * world
    for r in range(world):
        be = CudaRowShard(p, recs[r * d0l * d1:(r + 1) * d0l * d1], d0, d1, rb, world, 0)
        own = range(r * B // world, (r + 1) * B // world)
        for s, b in enumerate(own):
            be.put_keys(s, clients[b].evks, clients[b].sk_rgsw)
        bes.append(be)

    def run(r):
        own = slice(r * B // world, (r + 1) * B // world)
        q = torch.from_numpy(qs[own].astype(np.uint32).view(np.int32)).cuda()
        slots = np.arange(B // world, dtype=np.int32)
        outs[r] = answer_row_sharded(bes[r], comm.view(r), q, slots, d0, d1).cpu().numpy().view(np.uint32)
        torch.cuda.synchronize()

    ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    got = np.concatenate(outs).astype(np.uint64).reshape(B, 2, po.ring.k, po.n)
    db = O.encode_database([r.tobytes() for r in recs], d0, d1, rb, po)
    want = O.answer_batch(qs, np.stack([c.evks for c in clients]), np.stack([c.sk_rgsw for c in clients]), db,
                          d0, d1, po)
    assert np.array_equal(got, want)


# ---------------------------------------------------------------------------
# column-sharded mode (the reference's SHARD_ALL_GATHER, src/cluster.py:350-440)

class OracleColShard:
    """Oracle compute for one column-shard rank (tests only)."""

    def __init__(self, po, db_pm_cols, d0, d1, n, clients_own):
        self.po, self.db, self.d0, self.d1, self.n = po, db_pm_cols, d0, d1, n
        self.clients = clients_own
        R = po.ring
        self.ct = 2 * R.k * R.n

    def _rs(self, x, *shape):
        R = self.po.ring
        return x.numpy().astype(np.uint64).reshape(*shape, 2, R.k, R.n)

    def expand(self, q_own, _slots):
        qs = self._rs(q_own, -1)
        leaves = O.expand(qs, np.stack([c.evks for c in self.clients]), self.d0, self.d1, self.po)
        rg = O.build_rgsw(leaves[:, self.d0:], np.stack([c.sk_rgsw for c in self.clients]), self.po)
        B = len(qs)
        rows = torch.from_numpy(leaves[:, :self.d0].reshape(B, self.d0, self.ct).astype(np.int64))
        return rows, torch.from_numpy(rg.reshape(B, rg.shape[1], rg.shape[2], self.ct).astype(np.int64))

    def rowsel_coltor(self, rows_all, rg_low):
        R = self.po.ring
        B = rows_all.shape[0]
        sel = O.rowsel(self._rs(rows_all, B, self.d0), self.db, R)
        rg = self._rs(rg_low, B, rg_low.shape[1], rg_low.shape[2])
        out = O.coltor(sel, rg, self.po) if rg_low.shape[1] else sel[:, 0]
        return torch.from_numpy(out.reshape(B, self.ct).astype(np.int64))

    def coltor(self, parts, rg_high):
        B = parts.shape[0]
        out = O.coltor(self._rs(parts, B, self.n), self._rs(rg_high, B, rg_high.shape[1], rg_high.shape[2]),
                       self.po)
        return torch.from_numpy(out.reshape(B, self.ct).astype(np.int64))


def _col_rank_main(rank, world, port, out_path):
    import torch.distributed as dist

    from paper_2604_04696_b200.cluster import CountingComm, TorchComm, answer_col_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    po = O.test_params()
    B = 2 * world
    recs, clients, _, qs = _material(po, B)
    db = O.encode_database(recs, D0, D1, RB, po)               # (d1, d0, kn)
    d1l = D1 // world
    db_local = np.ascontiguousarray(db[rank * d1l:(rank + 1) * d1l])
    own = slice(rank * B // world, (rank + 1) * B // world)
    be = OracleColShard(po, db_local, D0, D1, world, clients[own])
    q_own = torch.from_numpy(qs[own].astype(np.int64))
    cc = CountingComm(TorchComm())
    out = answer_col_sharded(be, cc, q_own, None, D0, D1)
    np.save(out_path + f".{rank}.npy", out.numpy())
    np.save(out_path + f".ledger.{rank}.npy", np.array([cc.ledger.after_expand_bytes, cc.ledger.after_coltor_bytes,
                                                         cc.ledger.rgsw_sidecar_bytes], dtype=np.int64))
    dist.barrier()
    dist.destroy_process_group()


def test_col_sharded_gloo_matches_single_process(tmp_path):
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    path = str(tmp_path / "resp")
    mp.start_processes(_col_rank_main, args=(world, port, path), nprocs=world, start_method="spawn", join=True)
    got = np.concatenate([np.load(path + f".{r}.npy") for r in range(world)]).astype(np.uint64)
    po = O.test_params()
    B = 2 * world
    _check_ledger(path, world, "col", po, B)
    recs, clients, targets, qs = _material(po, B)
    db = O.encode_database(recs, D0, D1, RB, po)
    want = O.answer_batch(qs, np.stack([c.evks for c in clients]), np.stack([c.sk_rgsw for c in clients]), db,
                          D0, D1, po)
    assert np.array_equal(got.reshape(want.shape), want)
    for c, (i, j), ct in zip(clients, targets, want):
        assert O.decode_plain(O.decrypt(c, ct), RB, po) == recs[i * D1 + j]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_col_sharded_gpu_virtual_ranks(world):
    from paper_2604_04696_b200.cluster import CudaColShard, answer_col_sharded
    from tests.helpers import to_api

    po = O.default_params(plain_bits=16)
    p = to_api(po)
    d0, d1, rb = 16, 8, 1024
    B = 2 * world
    rng = np.random.default_rng(78)
    recs = rng.integers(0, 256, size=(d0 * d1, rb), dtype=np.uint8)
    clients = [O.client_keygen(po, d0, d1, rng) for _ in range(B)]
    targets = [(int(rng.integers(0, d0)), int(rng.integers(0, d1))) for _ in range(B)]
    qs = np.stack([O.client_query(c, i, j, d0, d1, rng) for c, (i, j) in zip(clients, targets)])
    comm = _ThreadComm(world)
    d1l = d1 // world
    grid = recs.reshape(d0, d1, rb)
    bes, outs = [], [None] * world
    for r in range(world):
        cols = np.ascontiguousarray(grid[:, r * d1l:(r + 1) * d1l]).reshape(d0 * d1l, rb)
        be = CudaColShard(p, cols, d0, d1, rb, world, 0)
        own = range(r * B // world, (r + 1) * B // world)
        for s, b in enumerate(own):
            be.put_keys(s, clients[b].evks, clients[b].sk_rgsw)
        bes.append(be)

    def run(r):
        own = slice(r * B // world, (r + 1) * B // world)
        q = torch.from_numpy(qs[own].astype(np.uint32).view(np.int32)).cuda()
        slots = np.arange(B // world, dtype=np.int32)
        outs[r] = answer_col_sharded(bes[r], comm.view(r), q, slots, d0, d1).cpu().numpy().view(np.uint32)
        torch.cuda.synchronize()

    ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    got = np.concatenate(outs).astype(np.uint64).reshape(B, 2, po.ring.k, po.n)
    db = O.encode_database([r.tobytes() for r in recs], d0, d1, rb, po)
    want = O.answer_batch(qs, np.stack([c.evks for c in clients]), np.stack([c.sk_rgsw for c in clients]), db,
                          d0, d1, po)
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_col_sharded_gpu_windows_compact():
    """Column shards held compact (byte planes only) with the shard's RowSel + low
    ColTor run per column window (gpir_sharded_rowsel_coltor) on 2 virtual ranks."""
    from paper_2604_04696_b200 import _native as nat
    from paper_2604_04696_b200.cluster import CudaColShard, answer_col_sharded
    from tests.helpers import to_api

    po = O.test_params()
    p = to_api(po)
    d0, d1, rb, world = 32, 128, 32, 2
    B = 4
    rng = np.random.default_rng(79)
    recs = rng.integers(0, 256, size=(d0 * d1, rb), dtype=np.uint8)
    clients = [O.client_keygen(po, d0, d1, rng) for _ in range(B)]
    targets = [(int(rng.integers(0, d0)), int(rng.integers(0, d1))) for _ in range(B)]
    qs = np.stack([O.client_query(c, i, j, d0, d1, rng) for c, (i, j) in zip(clients, targets)])
    comm = _ThreadComm(world)
    d1l = d1 // world
    grid = recs.reshape(d0, d1, rb)
    bes, outs = [], [None] * world
    R = po.ring
    for r in range(world):
        cols = torch.from_numpy(np.ascontiguousarray(grid[:, r * d1l:(r + 1) * d1l]).reshape(d0 * d1l, rb)).cuda()
        be = CudaColShard(p, cols, d0, d1, rb, world, 0, compact=True)
        nat.check(be.ctx.lib.gpir_set_capacity(be.ctx.h, B * 32 * 2 * R.k * R.n * 4, 0), "capacity")  # 32-col windows
        own = range(r * B // world, (r + 1) * B // world)
        for s_, b in enumerate(own):
            be.put_keys(s_, clients[b].evks, clients[b].sk_rgsw)
        bes.append(be)

    def run(r):
        own = slice(r * B // world, (r + 1) * B // world)
        q = torch.from_numpy(qs[own].astype(np.uint32).view(np.int32)).cuda()
        slots = np.arange(B // world, dtype=np.int32)
        outs[r] = answer_col_sharded(bes[r], comm.view(r), q, slots, d0, d1).cpu().numpy().view(np.uint32)
        torch.cuda.synchronize()

    ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    got = np.concatenate(outs).astype(np.uint64).reshape(B, 2, R.k, R.n)
    db = O.encode_database([r.tobytes() for r in recs], d0, d1, rb, po)
    want = O.answer_batch(qs, np.stack([c.evks for c in clients]), np.stack([c.sk_rgsw for c in clients]), db,
                          d0, d1, po)
    assert np.array_equal(got, want)
