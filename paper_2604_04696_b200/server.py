"""Batch collector in front of the GPU pipeline (the server step before the
hot path; mirrors latpir.server's batching, src/server.py:264-306).

The reference's connection threads deserialize every query into Python
objects, append them to a pending list, and a collector thread cuts a batch
when `batch_max` queries are pending or `batch_wait_ms` elapsed since the
first pending one (src/server.py:264-281); `_serve_batch` then restacks the
objects into the batch tensor and serialises each response.  Here the pending
list holds the framed bytes; a batch is decoded by ONE native call straight
into a page-locked (B, 2, k, n) buffer (`wire.decode_queries`), served by
`protocol.answer_raw` (gpir_answer_batch), and the framed responses are
encoded by ONE native call.  Message dispatch (`handle_message`) follows the
reference's `_conn_loop` (params request, key-set upload, queries, error
replies with the same codes).  The TCP transport itself stays out of scope:
callers hand in message bytes and a reply callback.
"""
from __future__ import annotations

import struct
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import planner, protocol, wire
from .errors import ParseError, PirError

_ERR = struct.Struct("<H")
_PARAMS_BODY = struct.Struct("<IBBBHHIII")  # n, k, plain_bits, z_bits, ell, err_bound, d0, d1, record_bytes


def serialize_error(code: int, message: str) -> bytes:
    """KIND_ERROR (src/wire.py:343-345)."""
    return wire._frame(wire.KIND_ERROR, _ERR.pack(code) + message.encode())


def deserialize_error(buf: bytes) -> tuple[int, str]:
    kind, _ = wire.parse_header(buf)
    if kind != wire.KIND_ERROR:
        raise ParseError(f"expected error message, got kind {kind}", 6)
    (code,) = _ERR.unpack_from(buf, wire.HEADER_BYTES)
    return code, buf[wire.HEADER_BYTES + 2:].decode(errors="replace")


def serialize_params(params, config) -> bytes:
    """KIND_PARAMS server profile (src/wire.py:321-329)."""
    body = _PARAMS_BODY.pack(params.n, params.basis.k, params.plain_bits, params.gadget.z_bits, params.gadget.ell,
                             params.error_bound, config.d0, config.d1, config.record_bytes)
    qs = b"".join(struct.pack("<Q", m.q) for m in params.basis.moduli)
    return wire._frame(wire.KIND_PARAMS, body + qs)


@dataclass
class CollectorConfig:
    """The batching knobs of latpir.server.ServerConfig (src/server.py:41-62)."""

    batch_max: int = 32
    batch_wait_ms: int = 50
    engine: str = "auto"


class BatchCollector:
    """Thread-safe batch former + GPU dispatch.  `submit(msg, reply)` queues a
    framed message; `reply(bytes)` is called with the framed response (or error)."""

    def __init__(self, db, params, config: CollectorConfig | None = None):
        self.db = db
        self.params = params
        self.config = config or CollectorConfig()
        self.keys: dict[int, object] = {}
        self.keys_lock = threading.Lock()
        self.pending: list[tuple[bytes, object, float]] = []
        self.cond = threading.Condition()
        self.stop_event = threading.Event()
        self.batches_served = 0
        self.batch_sizes: list[int] = []
        total = planner.expansion_leaves(db.config.d0, db.config.d1, params.gadget.ell)
        self._stages = planner.num_expand_stages(total)
        self._pinned = None  # (B_max, 2, k, n) page-locked decode target
        self._thread: threading.Thread | None = None

    # -- lifecycle ----------------------------------------------------------
    def start(self) -> "BatchCollector":
        self._thread = threading.Thread(target=self._collect_loop, daemon=True, name="gpir-collect")
        self._thread.start()
        return self

    def stop(self) -> None:
        self.stop_event.set()
        with self.cond:
            self.cond.notify_all()
        if self._thread is not None:
            self._thread.join(timeout=5)

    def __enter__(self):
        return self.start()

    def __exit__(self, *exc):
        self.stop()

    # -- messages (src/server.py:222-253) -------------------------------------
    def handle_message(self, msg: bytes, reply) -> None:
        try:
            kind, _ = wire.parse_header(msg)
            if kind == wire.KIND_PARAMS:
                reply(serialize_params(self.params, self.db.config))
            elif kind == wire.KIND_EVKSET:
                cid, keys = wire.decode_evkset(msg, self.params, self._stages)
                with self.keys_lock:
                    self.keys[cid] = keys
            elif kind == wire.KIND_QUERY:
                self.submit(msg, reply)
            else:
                reply(serialize_error(2, f"unexpected message kind {kind}"))
        except ParseError as exc:
            reply(serialize_error(1, str(exc)))

    def submit(self, msg: bytes, reply) -> None:
        with self.cond:
            self.pending.append((msg, reply, time.monotonic()))
            self.cond.notify_all()

    # -- batching (src/server.py:264-281) -------------------------------------
    def _collect_loop(self) -> None:
        wait_s = self.config.batch_wait_ms / 1000.0
        while not self.stop_event.is_set():
            with self.cond:
                while not self.pending and not self.stop_event.is_set():
                    self.cond.wait(timeout=0.1)
                if self.stop_event.is_set():
                    return
                deadline = self.pending[0][2] + wait_s
                while (len(self.pending) < self.config.batch_max and time.monotonic() < deadline
                       and not self.stop_event.is_set()):
                    self.cond.wait(timeout=max(deadline - time.monotonic(), 0.001))
                batch = self.pending[: self.config.batch_max]
                del self.pending[: len(batch)]
            if batch:
                self.serve_batch(batch)

    def _decode_target(self, B: int):
        b = self.params.basis
        if self._pinned is None or self._pinned.shape[0] < B:
            try:
                self._pinned = wire.pinned_queries(max(B, self.config.batch_max), b.k, b.n)
            except Exception:  # no CUDA host allocator: pageable buffer
                self._pinned = np.empty((max(B, self.config.batch_max), 2, b.k, b.n), dtype=np.uint32)
        return self._pinned

    def serve_batch(self, batch) -> None:
        """Decode -> GPU -> encode for one batch of (msg, reply[, t]) entries."""
        msgs = [e[0] for e in batch]
        replies = [e[1] for e in batch]
        b = self.params.basis
        good, bad = [], []
        try:
            qarr, ids, seqs = wire.decode_queries(msgs, b.n, b.k, out=self._decode_target(len(msgs)))
            good = list(range(len(msgs)))
        except ParseError:  # isolate the malformed messages, serve the rest
            for i, m in enumerate(msgs):
                try:
                    wire.decode_queries([m], b.n, b.k)
                    good.append(i)
                except ParseError as exc:
                    bad.append((i, exc))
            for i, exc in bad:
                replies[i](serialize_error(1, str(exc)))
            if not good:
                return
            qarr, ids, seqs = wire.decode_queries([msgs[i] for i in good], b.n, b.k,
                                                  out=self._decode_target(len(good)))
        with self.keys_lock:
            keys = dict(self.keys)
        try:
            out = protocol.answer_raw(qarr, ids, keys, self.db, self.params, engine=self.config.engine)
        except PirError as exc:  # report per query rather than dying (src/server.py:287-292)
            for i in good:
                replies[i](serialize_error(3, f"batch failed: {exc}"))
            return
        for i, m in zip(good, wire.encode_responses(out, ids, seqs)):
            replies[i](m)
        self.batches_served += 1
        self.batch_sizes.append(len(good))
