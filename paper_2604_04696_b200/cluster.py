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
350-440).  The row split shards every phase by n (expansion and ColTor by
query, RowSel by row), but its combine moves the partial selection of every
query and column: the reduce-scatter is (n-1)/n x B x d1 ciphertexts per rank,
which grows with the DB (56 GiB per rank at config 4, n = 8; `device_comm_bytes`).
The column split (`answer_col_sharded`) exchanges B x d0 row ciphertexts
(all-gather) plus B x n partial ciphertexts, independent of d1: it is the mode
for DBs that do not fit one GPU (configs 4-5), the row split the one for
DBs that do (configs 1-3, the north star's).

The orchestration is backend- and transport-agnostic so the exchange logic is
tested on CPU with gloo and the oracle backend (tests/test_cluster.py);
`CudaRowShard` / `CudaColShard` are the product backends, `TorchComm` the NCCL
transport and `CountingComm` the byte ledger of a run (reference:
CommLedger / comm_bytes, src/cluster.py:83-141).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from dataclasses import dataclass, field
from enum import Enum

from . import _native as nat
from .errors import InvalidArgument
from .protocol import Context, EncodedDatabase


class Strategy(Enum):
    """Multi-worker strategies: the reference's three (src/cluster.py:40-43)
    plus the north star's row split."""
    NAIVE_BATCH = "naive"
    SHARD_AGGREGATE = "shard_aggregate"
    SHARD_ALL_GATHER = "shard_all_gather"
    ROW_SHARD = "row_shard"


@dataclass
class CommLedger:
    """Byte counters for the two synchronization points (src/cluster.py:83-121):
    after expansion (row ciphertexts) and after the local tournament / RowSel
    (partials), plus the RGSW sidecar of the all-gather strategy."""

    after_expand_bytes: int = 0
    after_coltor_bytes: int = 0
    rgsw_sidecar_bytes: int = 0
    per_link: dict = field(default_factory=dict, compare=False)

    def add(self, phase: str, worker: int, nbytes: int) -> None:
        if phase == "expand":
            self.after_expand_bytes += nbytes
        elif phase == "coltor":
            self.after_coltor_bytes += nbytes
        else:
            self.rgsw_sidecar_bytes += nbytes
        key = (worker, phase)
        self.per_link[key] = self.per_link.get(key, 0) + nbytes

    def modeled_seconds(self, link_bandwidth: float) -> dict:
        if link_bandwidth <= 0:
            raise InvalidArgument("link bandwidth must be positive")
        return {"after_expand": self.after_expand_bytes / link_bandwidth,
                "after_coltor": self.after_coltor_bytes / link_bandwidth}

    def to_text(self, strategy: Strategy, n_workers: int, link_bandwidth: float | None = None) -> str:
        rows = [("after_expand", self.after_expand_bytes), ("after_coltor", self.after_coltor_bytes)]
        lines = ["strategy\tn_workers\tphase\tbytes\tmodeled_seconds"]
        for phase, nbytes in rows:
            modeled = f"{nbytes / link_bandwidth:.9f}" if link_bandwidth else "-"
            lines.append(f"{strategy.value}\t{n_workers}\t{phase}\t{nbytes}\t{modeled}")
        return "\n".join(lines) + "\n"


def comm_bytes(strategy: Strategy, config, batch: int, n_workers: int, params) -> CommLedger:
    """The reference's closed-form ledger in wire bytes (src/cluster.py:124-136):
    after_coltor = B n ct; the all-gather strategy adds after_expand = B d0 ct and
    the RGSW sidecar."""
    from . import wire

    led = CommLedger()
    if n_workers <= 1 or strategy in (Strategy.NAIVE_BATCH,):
        return led
    ct = wire.serialized_ct_bytes(params)
    if strategy is Strategy.ROW_SHARD:
        return device_comm_bytes(strategy, config, batch, n_workers, params)
    led.after_coltor_bytes = batch * n_workers * ct
    if strategy is Strategy.SHARD_ALL_GATHER:
        led.after_expand_bytes = batch * config.d0 * ct
        body = 6 + 2 * params.basis.k * params.n * 4
        led.rgsw_sidecar_bytes = batch * (config.d1.bit_length() - 1) * (wire.HEADER_BYTES + 3 + 2 * params.gadget.ell * body)
    return led


def device_comm_bytes(strategy: Strategy, config, batch: int, n_workers: int, params) -> CommLedger:
    """Bytes the NCCL collectives of this package move between ranks (sum over
    receiving ranks; a ciphertext is 2 k n u32 words on the device):
      ROW_SHARD: all-to-all of row blocks (n-1) B d0/n cts, reduce-scatter of the
                 partial selections (n-1) B d1 cts (it grows with the DB);
      SHARD_ALL_GATHER: all-gather of row cts (n-1) B d0, of the low-bit RGSW rows
                 (n-1) B log2(d1/n) 2 ell, all-to-all of partials (n-1)/n B n cts."""
    led = CommLedger()
    n = n_workers
    if n <= 1 or strategy in (Strategy.NAIVE_BATCH, Strategy.SHARD_AGGREGATE):
        return led
    ct = 2 * params.basis.k * params.n * 4
    B, d0, d1 = batch, config.d0, config.d1
    if strategy is Strategy.ROW_SHARD:
        led.after_expand_bytes = (n - 1) * B * (d0 // n) * ct
        led.after_coltor_bytes = (n - 1) * B * d1 * ct
    else:
        low = (d1 // n).bit_length() - 1
        led.after_expand_bytes = (n - 1) * B * d0 * ct
        led.rgsw_sidecar_bytes = (n - 1) * B * low * 2 * params.gadget.ell * ct
        led.after_coltor_bytes = (n - 1) * B * ct
    return led


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
    mark = getattr(comm, "mark", lambda phase: None)
    send = backend.swap01(rows.reshape(b_own, n, d0l, ct))  # (n, B_own, d0/n, CT)
    mark("expand")
    recv = comm.all_to_all(send)                      # recv[s] = rank s's queries, my row range
    partial = backend.rowsel(recv.reshape(n * b_own, d0l, ct))
    mark("coltor")
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
    mark = getattr(comm, "mark", lambda phase: None)
    rows, rgsw = backend.expand(queries_own, slots_own)
    b_own = rows.shape[0]
    mark("expand")
    rows_all = comm.all_gather(rows)                       # (n, B_own, d0, CT), rank order = query order
    if low:
        mark("rgsw")
        rg_low = comm.all_gather(rgsw[:, :low].contiguous())  # (n, B_own, low, 2 ELL, CT)
    else:
        rg_low = rgsw[:, :0].unsqueeze(0).expand((n,) + tuple(rgsw[:, :0].shape)).contiguous()
    part = backend.rowsel_coltor(rows_all.reshape((n * b_own,) + tuple(rows.shape[1:])),
                                 rg_low.reshape((n * b_own,) + tuple(rg_low.shape[2:])))
    mark("coltor")
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
        except (RuntimeError, NotImplementedError, ValueError):
            # backends without reduce_scatter (gloo): block r of every rank to rank r
            # (the same (n-1)/n volume), summed there
            recv = self.all_to_all(x.contiguous())
            out.copy_(recv.sum(dim=0, dtype=x.dtype))
        return out


class CountingComm:
    """Transport wrapper recording the bytes every rank receives from the others
    into a CommLedger (the measured side of `device_comm_bytes`).  The phase of
    each collective follows the orchestration: the first exchange of a batch is
    the row ciphertexts ("expand"), an all-gather of RGSW rows the sidecar, the
    last exchange the partials ("coltor")."""

    def __init__(self, comm, ledger: CommLedger | None = None):
        self.comm = comm
        self.size = comm.size
        self.rank = getattr(comm, "rank", 0)
        self.ledger = ledger if ledger is not None else CommLedger()
        self.phase = "expand"

    def mark(self, phase: str) -> None:
        """The orchestration names the synchronization point of the next exchange."""
        self.phase = phase

    def _count(self, nbytes_foreign: int):
        self.ledger.add(self.phase, self.rank, int(nbytes_foreign))

    def all_to_all(self, send):
        out = self.comm.all_to_all(send)
        self._count(send.element_size() * send.numel() * (self.size - 1) // self.size)
        return out

    def all_gather(self, x):
        out = self.comm.all_gather(x)
        self._count(x.element_size() * x.numel() * (self.size - 1))
        return out

    def reduce_scatter_sum(self, x):
        out = self.comm.reduce_scatter_sum(x)
        self._count(x.element_size() * x.numel() * (self.size - 1) // self.size)
        return out


def _encode_shard(ctx, params, recs, cfg, record_bytes: int, compact: bool):
    """Encode one rank's record shard: a (records, record_bytes) uint8 numpy array
    (host) or torch CUDA tensor (gpir_db_encode_dev); compact keeps only the
    RowSel byte planes."""
    if hasattr(recs, "is_cuda") and recs.is_cuda:
        if tuple(recs.shape) != (cfg.records, record_bytes):
            raise InvalidArgument(f"shard shape {tuple(recs.shape)} != {(cfg.records, record_bytes)}")
        import torch
        torch.cuda.synchronize(recs.device)
        h = ctx.lib.gpir_db_encode_dev(ctx.h, C.c_void_p(recs.data_ptr()), cfg.d0, cfg.d1, record_bytes,
                                       params.plain_bits)
    else:
        recs = np.ascontiguousarray(recs, dtype=np.uint8)
        if recs.shape != (cfg.records, record_bytes):
            raise InvalidArgument(f"shard shape {recs.shape} != {(cfg.records, record_bytes)}")
        h = ctx.lib.gpir_db_encode(ctx.h, nat.ptr(recs, C.c_uint8), cfg.d0, cfg.d1, record_bytes, params.plain_bits)
    if not h:
        raise nat.NativeError(f"gpir_db_encode failed: {nat.last_error()}")
    db = EncodedDatabase(cfg, params, ctx, h)
    return db.compact() if compact else db


class CudaRowShard:
    """Product backend: libgpir row-sharded entry points on this rank's GPU.

    `db_rows` is this rank's (d0/n, d1) slice of the record grid (uint8
    array, row-major records); queries/keys are uploaded per call."""

    def __init__(self, params, db_rows, d0: int, d1: int, record_bytes: int, n: int, device: int,
                 compact: bool = False):
        import torch

        from .values import DbConfig

        self.torch = torch
        self.params = params
        self.d0, self.d1, self.n = d0, d1, n
        self.device = device
        # a private context: the sharded session state (expand -> coltor) is per rank
        self.ctx = Context(params, device)
        cfg = DbConfig(d0 // n, d1, record_bytes)
        self.db = _encode_shard(self.ctx, params, db_rows, cfg, record_bytes, compact)
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

    def __init__(self, params, db_cols, d0: int, d1: int, record_bytes: int, n: int, device: int,
                 compact: bool = False):
        import torch

        from .values import DbConfig

        self.torch = torch
        self.params = params
        self.d0, self.d1, self.n = d0, d1, n
        self.device = device
        self.ctx = Context(params, device)
        cfg = DbConfig(d0, d1 // n, record_bytes)
        self.db = _encode_shard(self.ctx, params, db_cols, cfg, record_bytes, compact)
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
        # RowSel against this shard's columns + its low ColTor stages in one call
        # (per column window when the shard's selection exceeds the budget)
        lib, h = self.ctx.lib, self.ctx.h
        B = rows_all.shape[0]
        out = self._new(B, self.ct)
        rg = C.c_void_p(rgsw_low.data_ptr()) if rgsw_low.numel() else None
        nat.check(lib.gpir_sharded_rowsel_coltor(h, self.db.handle, C.c_void_p(rows_all.data_ptr()), B, rg,
                                                 C.c_void_p(out.data_ptr()), self._sp()), "sharded rowsel+coltor")
        return out

    def coltor(self, parts, rgsw_high):
        b_own = parts.shape[0]
        out = self._new(b_own, self.ct)
        nat.check(self.ctx.lib.gpir_coltor_dev(self.ctx.h, C.c_void_p(parts.data_ptr()), b_own, self.n,
                                               C.c_void_p(rgsw_high.data_ptr()), C.c_void_p(out.data_ptr()),
                                               self._sp()), "owner coltor")
        return out
