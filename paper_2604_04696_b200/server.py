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


# ---------------------------------------------------------------------------
# benchmark harness (latpir.server.run_bench / BenchReport, src/server.py:371-455)

_PHASES = ("ExpandQuery", "RgswAssembly", "RowSel", "ColTor")
_MODES = {0: "op", 1: "stage", 2: "split", 3: "stage"}


@dataclass
class BenchReport:
    """Same fields and text/CSV formats as the reference's BenchReport; the
    per-stage rows are measured on the GPU (CUDA events per stage) and
    `allocator_traffic_bytes` is the device workspace of the batch."""

    batch: int
    batches: int
    phase_ms_per_query: dict
    qps: float
    allocator_traffic_bytes: int
    stage_rows: list  # (phase, stage, nodes, working_set, mode, amortized_ms)
    plan_text: str
    ledger_text: str = ""

    def to_text(self) -> str:
        lines = [f"batch\t{self.batch}", f"batches\t{self.batches}", f"qps\t{self.qps:.3f}",
                 f"allocator_traffic_bytes\t{self.allocator_traffic_bytes}"]
        for phase, ms in self.phase_ms_per_query.items():
            lines.append(f"amortized_ms\t{phase}\t{ms:.3f}")
        lines.append("-- plan --")
        lines.append(self.plan_text.rstrip("\n"))
        if self.ledger_text:
            lines.append("-- comm --")
            lines.append(self.ledger_text.rstrip("\n"))
        return "\n".join(lines) + "\n"

    def stage_csv(self) -> str:
        rows = ["phase,stage,nodes,working_set_bytes,mode,amortized_ms"]
        for phase, stage, nodes, ws, mode, ms in self.stage_rows:
            rows.append(f"{phase},{stage},{nodes},{ws},{mode},{ms:.4f}")
        return "\n".join(rows) + "\n"


def run_bench(db, params, batches: int, batch: int = 32, seed: int = 1234, hw=None) -> BenchReport:
    """Serve `batches` seeded batches of `batch` queries and report amortized
    per-phase and per-stage costs (src/server.py:409-455).  Key and query
    material is uniform random (the kernels are data-oblivious), one key set per
    query slot; timing is device time from CUDA events."""
    import ctypes as C

    from . import _native as nat
    from .planner import HardwareModel, Phase, build_plan, working_set

    hw = hw or HardwareModel.b200()
    rng = np.random.default_rng(seed)
    b = params.basis
    k, n, ell = b.k, b.n, params.gadget.ell
    cfg = db.config
    stages = planner.num_expand_stages(planner.expansion_leaves(cfg.d0, cfg.d1, ell))
    qs = np.array([m.q for m in b.moduli], dtype=np.uint64)[:, None]

    def uni(*shape):
        return (rng.integers(0, 1 << 62, size=shape + (k, n), dtype=np.uint64) % qs).astype(np.uint32)

    from .wire import RawKeys

    keys = {c: RawKeys(n, uni(stages, ell, 2), uni(2 * ell, 2)) for c in range(batch)}
    ddb = protocol._device_db(db, params)
    ctx = ddb.ctx
    nat.check(ctx.lib.gpir_set_stage_timing(ctx.h, 1), "stage timing")
    plan = build_plan(cfg, params, batch, hw)
    phase_tot = {p: 0.0 for p in _PHASES}
    stage_acc: dict = {}
    wall = 0.0
    buf = (nat.GpirStageTime * 64)()
    try:
        for _ in range(batches):
            qarr = uni(batch, 2)
            t0 = time.perf_counter()
            protocol.answer_raw(qarr, list(range(batch)), keys, db, params, hw=hw, plan=plan)
            wall += time.perf_counter() - t0
            cnt = ctx.lib.gpir_stage_times(ctx.h, buf, len(buf))
            for e in buf[:min(cnt, len(buf))]:
                phase = _PHASES[e.phase]
                phase_tot[phase] += e.ms / 1e3
                if phase == "RowSel":
                    continue
                ph = Phase.EXPAND_QUERY if phase == "ExpandQuery" else Phase.COL_TOR
                ws = working_set(ph, e.stage, batch, params, cfg) if phase != "RgswAssembly" else 0
                key = (phase, e.stage, e.units // batch if phase != "RgswAssembly" else e.units, ws,
                       _MODES.get(e.mode, "op"))
                stage_acc.setdefault(key, []).append(e.ms / 1e3)
    finally:
        ctx.lib.gpir_set_stage_timing(ctx.h, 0)
    nq = batches * batch
    return BenchReport(
        batch=batch, batches=batches, phase_ms_per_query={p: t / nq * 1e3 for p, t in phase_tot.items()},
        qps=nq / wall if wall else 0.0, allocator_traffic_bytes=int(ddb.device_bytes),
        stage_rows=sorted(key + (sum(v) / nq * 1e3,) for key, v in stage_acc.items()),
        plan_text=plan.to_text() if hasattr(plan, "to_text") else str(plan))
