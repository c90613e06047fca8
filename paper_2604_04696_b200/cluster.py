"""Multi-GPU serving: the database row-sharded (north star) or column-sharded
(the reference's SHARD_ALL_GATHER) across ranks, one process per GPU.

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


def answer_col_sharded(backend, comm, queries_own, slots_own, d0: int, d1: int):
    """Column-sharded serving (the reference's SHARD_ALL_GATHER strategy,
    src/cluster.py:350-440, with NCCL collectives instead of worker threads).

    Rank r of n owns DB columns [r d1/n, (r+1) d1/n) x all d0 rows and the
    queries [r B/n, (r+1) B/n).
      1. every rank expands its OWN queries over the full tree and assembles
         their RGSWs;
      2. all-gather of the row ciphertexts (B x d0 cts; the reference's
         after_expand volume) and of the low-bit RGSW rows (its sidecar);
      3. local RowSel over the rank's columns for all B queries and the low
         log2(d1/n) ColTor stages -> one partial ciphertext per query;
      4. all-to-all of the partials to the query owners (the reference's
         after_coltor volume, B x n cts);
      5. the owner finishes the top log2(n) ColTor stages.
    The exchange volume does not depend on d1, so it scales with the DB.

    backend: .expand(queries_own, slots_own) -> (rows (B_own, d0, CT), rgsw (B_own, bits, 2 ELL, CT))
             .rowsel_coltor(rows_all (B, d0, CT), rgsw_low (B, low, 2 ELL, CT)) -> (B, CT)
             .coltor(parts (B_own, n, CT), rgsw_high (B_own, bits - low, 2 ELL, CT)) -> (B_own, CT)
    comm:    .size, .all_gather(x) -> (n, *x.shape), .all_to_all(send (n, ...)) -> (n, ...)
    """
    n = comm.size
    if d1 % n or (n & (n - 1)):
        raise InvalidArgument(f"d1={d1} does not split into {n} power-of-two column shards")
    low = (d1 // n).bit_length() - 1
    rows, rgsw = backend.expand(queries_own, slots_own)
    b_own = rows.shape[0]
    rows_all = comm.all_gather(rows)                       # (n, B_own, d0, CT), rank order = query order
    if low:
        rg_low = comm.all_gather(rgsw[:, :low].contiguous())  # (n, B_own, low, 2 ELL, CT)
    else:
        rg_low = rgsw[:, :0].unsqueeze(0).expand((n,) + tuple(rgsw[:, :0].shape)).contiguous()
    part = backend.rowsel_coltor(rows_all.reshape((n * b_own,) + tuple(rows.shape[1:])),
                                 rg_low.reshape((n * b_own,) + tuple(rg_low.shape[2:])))
    recv = comm.all_to_all(part.reshape((n, b_own) + tuple(part.shape[1:])))  # recv[s] = shard s's partials
    parts = recv.transpose(0, 1).contiguous()              # (B_own, n, CT): ct index = column shard
    return backend.coltor(parts, rgsw[:, low:].contiguous())


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

    def all_gather(self, x):
        import torch

        x = x.contiguous()
        out = torch.empty((self.size * x.shape[0],) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        self.dist.all_gather_into_tensor(out, x, group=self.group)  # concatenated along dim 0
        return out.view((self.size,) + tuple(x.shape))

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
        # torch's legacy default stream is handle 0, which the C ABI reads as "the
        # context's private stream"; pass cudaStreamLegacy (1) so the library's
        # launches stay ordered with the collectives torch queued on stream 0
        return C.c_void_p(self.stream.cuda_stream or 1)

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


class CudaColShard:
    """Product backend of `answer_col_sharded`: libgpir entry points on this
    rank's GPU.  `db_cols` holds this rank's column shard of the record grid as
    a (d0 * d1/n, record_bytes) uint8 array in row-major (i, j_local) order."""

    def __init__(self, params, db_cols: np.ndarray, d0: int, d1: int, record_bytes: int, n: int, device: int):
        import torch

        from .values import DbConfig

        self.torch = torch
        self.params = params
        self.d0, self.d1, self.n = d0, d1, n
        self.device = device
        self.ctx = Context(params, device)
        cfg = DbConfig(d0, d1 // n, record_bytes)
        recs = np.ascontiguousarray(db_cols, dtype=np.uint8)
        if recs.shape != (cfg.records, record_bytes):
            raise InvalidArgument(f"column shard shape {recs.shape} != {(cfg.records, record_bytes)}")
        h = self.ctx.lib.gpir_db_encode(self.ctx.h, nat.ptr(recs, C.c_uint8), cfg.d0, cfg.d1, record_bytes,
                                        params.plain_bits)
        if not h:
            raise nat.NativeError(f"gpir_db_encode failed: {nat.last_error()}")
        self.db = EncodedDatabase(cfg, params, self.ctx, h)
        b = params.basis
        self.k, self.nn, self.ell = b.k, b.n, params.gadget.ell
        self.ct = 2 * b.k * b.n
        self.bits = d1.bit_length() - 1
        self.stream = torch.cuda.current_stream(device)

    def _sp(self):
        # torch's legacy default stream is handle 0, which the C ABI reads as "the
        # context's private stream"; pass cudaStreamLegacy (1) so the library's
        # launches stay ordered with the collectives torch queued on stream 0
        return C.c_void_p(self.stream.cuda_stream or 1)

    def _new(self, *shape):
        return self.torch.empty(shape, dtype=self.torch.int32, device=f"cuda:{self.device}")

    def put_keys(self, slot: int, evks: np.ndarray, sk_rgsw: np.ndarray | None):
        ev = np.ascontiguousarray(evks, dtype=np.uint32)
        rg = None if sk_rgsw is None else np.ascontiguousarray(sk_rgsw, dtype=np.uint32)
        nat.check(self.ctx.lib.gpir_keys_put(self.ctx.h, slot, nat.ptr(ev), ev.shape[0], nat.ptr(rg)), "keys")

    def expand(self, queries_own, slots_own):
        lib, h = self.ctx.lib, self.ctx.h
        b_own = queries_own.shape[0]
        rows = self._new(b_own, self.d0, self.ct)
        nat.check(lib.gpir_sharded_expand(h, self.d0, self.d1, C.c_void_p(queries_own.data_ptr()),
                                          nat.ptr(slots_own, C.c_int32), b_own, C.c_void_p(rows.data_ptr()),
                                          self._sp()), "sharded expand")
        rg = self._new(b_own, self.bits, 2 * self.ell, self.ct)
        if self.bits:
            nat.check(lib.gpir_sharded_rgsw(h, 0, self.bits, C.c_void_p(rg.data_ptr()), self._sp()), "sharded rgsw")
        return rows, rg

    def rowsel_coltor(self, rows_all, rgsw_low):
        lib, h = self.ctx.lib, self.ctx.h
        B, d1l = rows_all.shape[0], self.d1 // self.n
        sel = self._new(B, d1l, self.ct)
        nat.check(lib.gpir_sharded_rowsel(h, self.db.handle, C.c_void_p(rows_all.data_ptr()), B,
                                          C.c_void_p(sel.data_ptr()), self._sp()), "sharded rowsel")
        nat_sel = self._new(B, d1l, self.ct)  # internal slot order -> natural for the tournament
        nat.check(lib.gpir_layout_convert(h, C.c_void_p(sel.data_ptr()), C.c_void_p(nat_sel.data_ptr()),
                                          B * d1l * 2, self._sp()), "layout")
        out = self._new(B, self.ct)
        nat.check(lib.gpir_coltor_dev(h, C.c_void_p(nat_sel.data_ptr()), B, d1l, C.c_void_p(rgsw_low.data_ptr()),
                                      C.c_void_p(out.data_ptr()), self._sp()), "local coltor")
        return out

    def coltor(self, parts, rgsw_high):
        b_own = parts.shape[0]
        out = self._new(b_own, self.ct)
        nat.check(self.ctx.lib.gpir_coltor_dev(self.ctx.h, C.c_void_p(parts.data_ptr()), b_own, self.n,
                                               C.c_void_p(rgsw_high.data_ptr()), C.c_void_p(out.data_ptr()),
                                               self._sp()), "owner coltor")
        return out
