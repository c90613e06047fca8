"""Multi-GPU serving: the database row-sharded across ranks (one process per GPU).

North-star mode: rank r of n owns DB rows
[r d0/n, (r+1) d0/n) x all d1 columns and the queries [r B/n, (r+1) B/n).

  1. every rank expands its OWN queries over the full tree and assembles their
     RGSWs (gpir_sharded_expand);
  2. all-to-all of row blocks: rank r receives, from every rank, that rank's
     queries' row ciphertexts of r's row range (B x d0/n cts in total);
  3. local RowSel over those rows (gpir_sharded_rowsel) -> partial sums for all
     B queries x d1 columns;
  4. reduce-scatter(sum) by query owner over NCCL: the modular-add combine of
     the RowSel partial accumulators (int32: n residues < 2^27 never wrap);
  5. the owner reduces mod q and runs the column tournament for its queries
     (gpir_sharded_coltor).

Bit-identical to one GPU: RowSel is a sum over rows, split exactly by rows,
and everything else runs on the query's owner with the same arithmetic.  The
reference's own multi-worker strategies shard columns (src/cluster.py:5-15,
350-440); the row split is the north star's, and it shards every phase by n
(expansion and ColTor by query, RowSel by row) with two collectives whose
volume does not grow with the DB.

The orchestration (`answer_row_sharded`) is backend- and transport-agnostic so
the exchange logic is tested on CPU with gloo and the oracle backend
(tests/test_cluster.py); `CudaRowShard` is the product backend and
`TorchComm` the NCCL transport.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .errors import InvalidArgument
from .protocol import Context, EncodedDatabase


def answer_row_sharded(backend, comm, queries_own, slots_own, d0: int, d1: int):
    """Run steps 1-5 for this rank; returns its own queries' responses.

    backend: .swap01(x) -> x with axes 0 and 1 exchanged (contiguous)
             .expand(queries_own, slots_own) -> rows (B_own, d0, CT)
             .rowsel(rows_all (B, d0/n, CT)) -> partial (B, d1, CT)
             .coltor(sums (B_own, d1, CT)) -> responses (B_own, CT)
    comm:    .size, .all_to_all(send (n, ...)) -> recv (n, ...),
             .reduce_scatter_sum(x (n, ...)) -> (...) block of this rank
    """
    n = comm.size
    if d0 % n:
        raise InvalidArgument(f"d0={d0} does not split over {n} ranks")
    rows = backend.expand(queries_own, slots_own)
    b_own = rows.shape[0]
    ct = rows.shape[-1]
    d0l = d0 // n
    send = backend.swap01(rows.reshape(b_own, n, d0l, ct))  # (n, B_own, d0/n, CT)
    recv = comm.all_to_all(send)                      # recv[s] = rank s's queries, my row range
    partial = backend.rowsel(recv.reshape(n * b_own, d0l, ct))
    sums = comm.reduce_scatter_sum(partial.reshape(n, b_own * d1 * ct))
    return backend.coltor(sums.reshape(b_own, d1, ct))


class TorchComm:
    """torch.distributed transport (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_to_all(self, send):
        import torch

        recv = torch.empty_like(send)
        self.dist.all_to_all_single(recv, send, group=self.group)
        return recv

    def reduce_scatter_sum(self, x):
        import torch

        out = torch.empty(x.shape[1:], dtype=x.dtype, device=x.device)
        try:
            self.dist.reduce_scatter_tensor(out, x, op=self.dist.ReduceOp.SUM, group=self.group)
        except (RuntimeError, NotImplementedError, ValueError):  # backends without reduce_scatter (gloo)
            y = x.clone()
            self.dist.all_reduce(y, op=self.dist.ReduceOp.SUM, group=self.group)
            out.copy_(y[self.rank])
        return out


class CudaRowShard:
    """Product backend: libgpir row-sharded entry points on this rank's GPU.

    `db_rows` is this rank's (d0/n, d1) slice of the record grid (uint8
    array, row-major records); queries/keys are uploaded per call."""

    def __init__(self, params, db_rows: np.ndarray, d0: int, d1: int, record_bytes: int, n: int, device: int):
        import torch

        from .values import DbConfig

        self.torch = torch
        self.params = params
        self.d0, self.d1, self.n = d0, d1, n
        self.device = device
        # a private context: the sharded session state (expand -> coltor) is per rank
        self.ctx = Context(params, device)
        cfg = DbConfig(d0 // n, d1, record_bytes)
        recs = np.ascontiguousarray(db_rows, dtype=np.uint8)
        if recs.shape != (cfg.records, record_bytes):
            raise InvalidArgument(f"row shard shape {recs.shape} != {(cfg.records, record_bytes)}")
        h = self.ctx.lib.gpir_db_encode(self.ctx.h, nat.ptr(recs, C.c_uint8), cfg.d0, cfg.d1, record_bytes,
                                        params.plain_bits)
        if not h:
            raise nat.NativeError(f"gpir_db_encode failed: {nat.last_error()}")
        self.db = EncodedDatabase(cfg, params, self.ctx, h)
        b = params.basis
        self.ct = 2 * b.k * b.n
        self.stream = torch.cuda.current_stream(device)

    def _sp(self):
        return C.c_void_p(self.stream.cuda_stream)

    def swap01(self, t):
        return t.transpose(0, 1).contiguous()

    def put_keys(self, slot: int, evks: np.ndarray, sk_rgsw: np.ndarray | None):
        """Upload one client's evks (stages, ell, 2, k, n) and RGSW(s) into key slot `slot`."""
        ev = np.ascontiguousarray(evks, dtype=np.uint32)
        rg = None if sk_rgsw is None else np.ascontiguousarray(sk_rgsw, dtype=np.uint32)
        nat.check(self.ctx.lib.gpir_keys_put(self.ctx.h, slot, nat.ptr(ev), ev.shape[0], nat.ptr(rg)), "keys")

    def expand(self, queries_own, slots_own):
        t = self.torch
        b_own = queries_own.shape[0]
        rows = t.empty((b_own, self.d0, self.ct), dtype=t.int32, device=f"cuda:{self.device}")
        nat.check(self.ctx.lib.gpir_sharded_expand(self.ctx.h, self.d0, self.d1, C.c_void_p(queries_own.data_ptr()),
                                                   nat.ptr(slots_own, C.c_int32), b_own, C.c_void_p(rows.data_ptr()),
                                                   self._sp()), "sharded expand")
        return rows

    def rowsel(self, rows_all):
        t = self.torch
        B = rows_all.shape[0]
        part = t.empty((B, self.d1, self.ct), dtype=t.int32, device=f"cuda:{self.device}")
        nat.check(self.ctx.lib.gpir_sharded_rowsel(self.ctx.h, self.db.handle, C.c_void_p(rows_all.data_ptr()), B,
                                                   C.c_void_p(part.data_ptr()), self._sp()), "sharded rowsel")
        return part

    def coltor(self, sums):
        t = self.torch
        b_own = sums.shape[0]
        out = t.empty((b_own, self.ct), dtype=t.int32, device=f"cuda:{self.device}")
        nat.check(self.ctx.lib.gpir_sharded_coltor(self.ctx.h, C.c_void_p(sums.data_ptr()), b_own,
                                                   C.c_void_p(out.data_ptr()), self._sp()), "sharded coltor")
        return out
