"""Drop-in server API: `encode_database`, `answer_batch`, `respond`.

Same signatures, argument meaning and error behaviour as the reference's
`latpir.protocol` (src/protocol.py:118-153, 635-688); the work runs in
libgpir.so on the GPU (include/gpir.h).  Inputs may be this package's value
types or the reference's own (duck-typed: `q.ct.a.limbs`, `keys.evk_raw`,
`params.basis.moduli`, ...); responses are built with the caller's classes so
the reference client can decode them unchanged.
"""
from __future__ import annotations

import sys
import threading
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import layout, planner
from .errors import InvalidArgument, InvalidState
from .planner import ExecMode, ExecutionPlan, HardwareModel, Phase
from .values import (
    BfvCiphertext,
    DbConfig,
    Domain,
    LayoutKind,
    Response,
    RnsPoly,
    U64,
    ct_from_raw,
)

# ---------------------------------------------------------------------------
# device context per (device, ring, gadget)


def _ring_key(params):
    b = params.basis
    return (tuple(int(m.q) for m in b.moduli), tuple(int(m.two_n_root) for m in b.moduli), int(b.n),
            int(params.gadget.z_bits), int(params.gadget.ell))


class Context:
    """Owns one gpir_ctx (tables, key pool, workspace) on one device."""

    def __init__(self, params, device: int = 0):
        self.lib = nat.load()
        qs, psis, n, zb, ell = _ring_key(params)
        self.n, self.k, self.ell, self.z_bits = n, len(qs), ell, zb
        self.device = device
        qa = np.array(qs, dtype=np.uint32)
        pa = np.array(psis, dtype=np.uint32)
        h = self.lib.gpir_ctx_create(device, n, len(qs), nat.ptr(qa), nat.ptr(pa), zb, ell)
        if not h:
            raise nat.NativeError(f"gpir_ctx_create failed: {nat.last_error()}")
        self.h = h
        self._slots: dict[int, tuple] = {}   # id(keys) -> (slot, weakref)
        self._free: list[int] = []
        self._next = 0
        # re-entrant: the weakref callback below may fire (GC) while this thread holds it
        self._lock = threading.RLock()

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.gpir_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # -- keys -----------------------------------------------------------------
    def key_slot(self, keys, stages: int, need_rgsw: bool) -> int:
        """Slot of a ClientKeys object, uploading it on first use (session-scoped)."""
        with self._lock:
            ent = self._slots.get(id(keys))
            if ent is not None and ent[1]() is keys and ent[2] >= stages and (ent[3] or not need_rgsw):
                return ent[0]
            if ent is not None and ent[1]() is keys:
                slot = ent[0]
            else:
                slot = self._free.pop() if self._free else self._next
                if slot == self._next:
                    self._next += 1
            evks = np.ascontiguousarray(
                np.stack([_evk_raw(keys, self.n // (1 << t) + 1) for t in range(stages)]).astype(np.uint32)
            ) if stages else None
            rg = None
            has_rg = False
            if need_rgsw or getattr(keys, "sk_rgsw", None) is not None:
                try:
                    rg = np.ascontiguousarray(_rgsw_raw(keys).astype(np.uint32))
                    has_rg = True
                except InvalidState:
                    if need_rgsw:
                        raise
            nat.check(self.lib.gpir_keys_put(self.h, slot, nat.ptr(evks), stages, nat.ptr(rg)), "keys upload")

            def _gone(_ref, slot=slot, key=id(keys), ctx=weakref.ref(self)):
                c = ctx()
                if c is not None and c.h:
                    # drop in C before the slot becomes reusable: a late drop would
                    # otherwise empty a slot another key set was just uploaded to
                    with c._lock:
                        ent = c._slots.get(key)
                        if ent is not None and ent[0] == slot:
                            c._slots.pop(key, None)
                        c.lib.gpir_keys_drop(c.h, slot)
                        c._free.append(slot)

            try:
                ref = weakref.ref(keys, _gone)
            except TypeError:  # not weak-referenceable: keep it alive with the slot
                ref = (lambda k=keys: k)
            self._slots[id(keys)] = (slot, ref, stages, has_rg)
            return slot


_contexts: dict = {}
_ctx_lock = threading.Lock()


def get_context(params, device: int | None = None) -> Context:
    if device is None:
        device = _current_device()
    key = (device,) + _ring_key(params)
    with _ctx_lock:
        ctx = _contexts.get(key)
        if ctx is None:
            ctx = Context(params, device)
            _contexts[key] = ctx
        return ctx


def _current_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return 0


def _evk_raw(keys, k_aut: int) -> np.ndarray:
    if hasattr(keys, "evk_raw"):
        return np.asarray(keys.evk_raw(k_aut))
    for e in keys.evks:
        if e.k_aut == k_aut:
            return np.stack([c.raw() for c in e.ksk])
    raise InvalidState(f"no evaluation key for automorphism index {k_aut}")


def _rgsw_raw(keys) -> np.ndarray:
    if hasattr(keys, "sk_rgsw_raw"):
        return np.asarray(keys.sk_rgsw_raw())
    if getattr(keys, "sk_rgsw", None) is None:
        raise InvalidState("this key set has no RGSW of the secret (onion mode needs one)")
    return keys.sk_rgsw.raw()


# ---------------------------------------------------------------------------
# database

class EncodedDatabase:
    """d0 x d1 NTT-encoded plaintexts resident in HBM (gpir_db).

    `data` materialises the reference's P-major (d1, d0, k*n) uint64 tensor on
    demand (src/protocol.py:64-99); the hot path never reads it."""

    def __init__(self, config: DbConfig, params, ctx: Context, handle, kind: LayoutKind = LayoutKind.P_MAJOR):
        self.config = config
        self.params = params
        self.ctx = ctx
        self.handle = handle
        self.layout = kind
        self._data = None
        self._owner = None

    def __del__(self):
        try:
            if self._owner is None and self.handle and self.ctx.h:
                self.ctx.lib.gpir_db_destroy(self.ctx.h, self.handle)
                self.handle = None
        except Exception:
            pass

    @property
    def raw_bytes(self) -> int:
        return self.config.records * self.config.record_bytes

    @property
    def encoded_bytes(self) -> int:
        return self.config.records * self.params.basis.k * self.params.basis.n * 4

    @property
    def device_bytes(self) -> int:
        return int(self.ctx.lib.gpir_db_bytes(self.handle))

    @property
    def data(self) -> np.ndarray:
        if self._data is None:
            b = self.params.basis
            out = np.empty((self.config.d1, self.config.d0, b.k * b.n), dtype=np.uint32)
            nat.check(self.ctx.lib.gpir_db_download(self.ctx.h, self.handle, nat.ptr(out)), "db download")
            pm = out.astype(U64)
            if self.layout is LayoutKind.TRANSPOSED:
                pm = np.ascontiguousarray(pm.transpose(2, 0, 1))
            self._data = pm
        return self._data

    def poly(self, i: int, j: int) -> RnsPoly:
        b = self.params.basis
        pm = self.data if self.layout is LayoutKind.P_MAJOR else self.data.transpose(1, 2, 0)
        return RnsPoly(b, pm[j, i].reshape(b.k, b.n).copy(), Domain.NTT)

    def compact(self) -> "EncodedDatabase":
        """Capacity mode (gpir_db_compact): keep only the tensor-core byte-plane
        image in HBM; `data` can no longer be downloaded."""
        nat.check(self.ctx.lib.gpir_db_compact(self.ctx.h, self.handle), "db compact")
        return self

    def to_layout(self, kind: LayoutKind) -> "EncodedDatabase":
        if kind is self.layout:
            return self
        other = EncodedDatabase(self.config, self.params, self.ctx, self.handle, kind)
        other._owner = self  # shares (and keeps alive) the device buffer
        return other


def encode_database(records, config: DbConfig, params, kind: LayoutKind = LayoutKind.P_MAJOR,
                    device: int | None = None) -> EncodedDatabase:
    """Pack records base-P, center mod P, lift mod Q and NTT them on the GPU
    (src/protocol.py:118-153)."""
    if params.plain_bits % 8 or params.plain_bits > 32:
        raise InvalidArgument("plaintext modulus must be a byte-aligned power of two up to 2**32")
    if params.plain_bits == 24:
        # the reference packs words with numpy '<u3', which does not exist (src/protocol.py:106-107)
        raise TypeError("data type '<u3' not understood")
    if config.record_bytes * 8 > params.basis.n * params.plain_bits:
        raise InvalidArgument("record does not fit one plaintext polynomial")
    if len(records) != config.records:
        raise InvalidArgument(f"expected {config.records} records, got {len(records)}")
    buf = np.zeros((config.records, config.record_bytes), dtype=np.uint8)
    for r, rec in enumerate(records):
        if len(rec) > config.record_bytes:
            raise InvalidArgument(f"record {r} exceeds {config.record_bytes} bytes")
        buf[r, :len(rec)] = np.frombuffer(bytes(rec), dtype=np.uint8)
    return encode_database_array(buf, config, params, kind, device)


def encode_database_array(buf: np.ndarray, config: DbConfig, params, kind: LayoutKind = LayoutKind.P_MAJOR,
                          device: int | None = None) -> EncodedDatabase:
    """Same as `encode_database` from a (records, record_bytes) uint8 array."""
    ctx = get_context(params, device)
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    if buf.shape != (config.records, config.record_bytes):
        raise InvalidArgument(f"record array shape {buf.shape} != {(config.records, config.record_bytes)}")
    h = ctx.lib.gpir_db_encode(ctx.h, nat.ptr(buf, nat.C.c_uint8), config.d0, config.d1, config.record_bytes,
                               params.plain_bits)
    if not h:
        raise nat.NativeError(f"gpir_db_encode failed: {nat.last_error()}")
    return EncodedDatabase(config, params, ctx, h, kind)


def encode_database_device(records, config: DbConfig, params, kind: LayoutKind = LayoutKind.P_MAJOR,
                           compact: bool = False) -> EncodedDatabase:
    """Same as `encode_database` from a torch uint8 tensor (records, record_bytes)
    already on the GPU (gpir_db_encode_dev): DBs of many GiB are generated and
    encoded on the device.  compact=True keeps only the RowSel byte-plane image."""
    import torch

    if records.dtype != torch.uint8 or not records.is_cuda or not records.is_contiguous():
        raise InvalidArgument("records must be a contiguous uint8 CUDA tensor")
    if tuple(records.shape) != (config.records, config.record_bytes):
        raise InvalidArgument(f"record tensor shape {tuple(records.shape)} != {(config.records, config.record_bytes)}")
    if config.record_bytes * 8 > params.basis.n * params.plain_bits:
        raise InvalidArgument("record does not fit one plaintext polynomial")
    ctx = get_context(params, records.device.index)
    torch.cuda.synchronize(records.device)
    h = ctx.lib.gpir_db_encode_dev(ctx.h, nat.C.c_void_p(records.data_ptr()), config.d0, config.d1,
                                   config.record_bytes, params.plain_bits)
    if not h:
        raise nat.NativeError(f"gpir_db_encode_dev failed: {nat.last_error()}")
    db = EncodedDatabase(config, params, ctx, h, kind)
    return db.compact() if compact else db


def upload_database(db, device: int | None = None) -> EncodedDatabase:
    """Move a reference-encoded database (numpy `data`) into HBM."""
    params, cfg = db.params, db.config
    ctx = get_context(params, device)
    data = np.asarray(db.data)
    if getattr(db.layout, "value", None) == "transposed":
        data = data.transpose(1, 2, 0)
    pm = np.ascontiguousarray(data, dtype=np.uint32)
    h = ctx.lib.gpir_db_upload(ctx.h, nat.ptr(pm), cfg.d0, cfg.d1)
    if not h:
        raise nat.NativeError(f"gpir_db_upload failed: {nat.last_error()}")
    return EncodedDatabase(cfg, params, ctx, h)


_uploaded: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _device_db(db, params) -> EncodedDatabase:
    if isinstance(db, EncodedDatabase):
        return db
    try:
        got = _uploaded.get(db)
    except TypeError:  # not weak-referenceable: upload without caching
        return upload_database(db)
    if got is None:
        got = upload_database(db)
        _uploaded[db] = got
    return got


# ---------------------------------------------------------------------------
# serving

@dataclass
class StageTiming:
    phase: str
    stage: int
    nodes: int
    mode: str
    working_set: int
    seconds: float
    peak_transient_bytes: int


@dataclass
class ServeStats:
    """Per-phase device seconds (CUDA events), as latpir.protocol.ServeStats."""

    phase_seconds: dict = field(default_factory=dict)
    stages: list = field(default_factory=list)
    arena_total_bytes: int = 0
    launches: int = 0
    h2d_seconds: float = 0.0
    d2h_seconds: float = 0.0
    device_seconds: float = 0.0

    def add_phase(self, name: str, seconds: float) -> None:
        self.phase_seconds[name] = self.phase_seconds.get(name, 0.0) + seconds


# every reference engine name is accepted (all give identical results); on the
# GPU "cudacore" / "pmajor" / "naive" pin the CUDA-core RowSel kernel and
# "tensorcore" the tcgen05 one, the rest choose automatically.
_ENGINES = {"auto": 0, "cuda": 0, "transposed": 0, "pipeline": 0, "pmajor": 1, "naive": 1, "cudacore": 1,
            "tensorcore": 2}


STAGE_CODE = 3


def _modes(config, params, B, hw, plan, mode):
    ell = params.gadget.ell
    total = planner.expansion_leaves(config.d0, config.d1, ell)
    ne, nc = planner.num_expand_stages(total), planner.num_coltor_stages(config.d1)
    # STAGE_LEVEL runs B200's stage-level executor (C-ABI mode 3: the digit
    # NTTs stream straight into the key-switch MAC, no materialised digit
    # NTTs), OPERATION_LEVEL the per-primitive kernels (mode 0)
    if mode is not None:
        v = STAGE_CODE if mode is ExecMode.STAGE_LEVEL or getattr(mode, "value", None) == "stage" else 0
        return np.full(max(ne, 1), v, np.uint8), np.full(max(nc, 1), v, np.uint8)
    if plan is None:
        plan = planner.build_plan(config, params, B, hw if hw is not None else HardwareModel.b200())
    fused = lambda m: STAGE_CODE if getattr(m, "value", m) == "stage" else 0
    em = np.array([fused(plan.mode_for(Phase.EXPAND_QUERY, t)) for t in range(ne)] or [0], np.uint8)
    cm = np.array([fused(plan.mode_for(Phase.COL_TOR, t)) for t in range(nc)] or [0], np.uint8)
    return em, cm


def _make_response(query, raw: np.ndarray):
    """Build the response with the caller's own classes (reference or ours)."""
    qct = query.ct
    poly_t, ct_t = type(qct.a), type(qct)
    a = poly_t(qct.a.basis, np.ascontiguousarray(raw[0].astype(U64)), qct.a.domain)
    b = poly_t(qct.a.basis, np.ascontiguousarray(raw[1].astype(U64)), qct.a.domain)
    mod = sys.modules.get(type(query).__module__)
    resp_t = getattr(mod, "Response", Response) if mod is not None else Response
    return resp_t(ct_t(a, b), query.client_id, query.seq)


def answer_raw(qarr: np.ndarray, client_ids, keys_by_client, db, params, hw: HardwareModel | None = None,
               plan: ExecutionPlan | None = None, mode: ExecMode | None = None, engine: str = "auto",
               stats: ServeStats | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """Serve a batch given as one (B, 2, k, n) uint32 array of NTT-domain query
    ciphertexts (natural slot order) and the per-query client ids; returns the
    (B, 2, k, n) responses.  This is the path the wire batch collector uses: the
    decoded bytes go straight in (pinned buffers avoid a staging copy)."""
    B = int(qarr.shape[0])
    if engine not in _ENGINES:
        raise InvalidArgument(f"unknown row-selection engine {engine!r}")
    config = db.config
    try:
        keys = [keys_by_client[int(c)] for c in client_ids]
    except KeyError as exc:
        raise InvalidState(f"no uploaded keys for client {exc.args[0]}") from None
    ddb = _device_db(db, params)
    ctx = ddb.ctx
    if qarr.shape != (B, 2, ctx.k, ctx.n) or qarr.dtype != np.uint32 or not qarr.flags.c_contiguous:
        raise InvalidArgument(f"queries must be a contiguous uint32 array of shape (B, 2, {ctx.k}, {ctx.n})")
    ell = params.gadget.ell
    total = planner.expansion_leaves(config.d0, config.d1, ell)
    stages = planner.num_expand_stages(total)
    need_rg = config.d1 > 1
    slots = np.array([ctx.key_slot(k, stages, need_rg) for k in keys], dtype=np.int32)
    em, cm = _modes(config, params, B, hw, plan, mode)
    if out is None:
        out = np.empty_like(qarr)
    nat.check(ctx.lib.gpir_set_rowsel_engine(ctx.h, _ENGINES[engine]), "rowsel engine")
    # per-phase events only when asked for: without them the library replays a
    # captured CUDA graph of the pipeline from the third call of a shape on
    st = nat.GpirStats() if stats is not None else None
    if stats is not None:  # per-stage CUDA events for ServeStats.stages
        nat.check(ctx.lib.gpir_set_stage_timing(ctx.h, 1), "stage timing")
    t0 = time.perf_counter()
    try:
        nat.check(ctx.lib.gpir_answer_batch(ctx.h, ddb.handle, nat.ptr(qarr), nat.ptr(slots, nat.C.c_int32), B,
                                            nat.ptr(em, nat.C.c_uint8), len(em), nat.ptr(cm, nat.C.c_uint8),
                                            len(cm), nat.ptr(out), nat.C.byref(st) if st is not None else None),
                  "answer_batch")
    finally:
        if stats is not None:
            ctx.lib.gpir_set_stage_timing(ctx.h, 0)
    wall = time.perf_counter() - t0
    if stats is not None:
        stats.add_phase(Phase.EXPAND_QUERY.value, st.ms_expand / 1e3)
        stats.add_phase("RgswAssembly", st.ms_rgsw / 1e3)
        stats.add_phase(Phase.ROW_SEL.value, st.ms_rowsel / 1e3)
        stats.add_phase(Phase.COL_TOR.value, st.ms_coltor / 1e3)
        stats.launches += st.launches
        stats.h2d_seconds += st.ms_h2d / 1e3
        stats.d2h_seconds += st.ms_d2h / 1e3
        stats.device_seconds += st.ms_total / 1e3
        stats.stages.extend(_stage_timings(ctx, config, params, B))
    return out


_PHASE_NAMES = {0: Phase.EXPAND_QUERY.value, 1: "RgswAssembly", 2: Phase.ROW_SEL.value, 3: Phase.COL_TOR.value}


def _stage_timings(ctx, config, params, B: int) -> list:
    """One StageTiming per ExpandQuery stage, RGSW assembly, RowSel and ColTor
    stage of the last batch (gpir_stage_times; src/protocol.py:301-320, 350-362).
    mode is the reference's ExecMode value of the executor ("op" / "stage");
    working_set the reference's transient-bytes model of the stage
    (planner.working_set) and peak_transient_bytes what the executor
    materialises in HBM: the working set for operation-level stages, 0 for
    stage-level ones (their digit NTTs stay on chip)."""
    buf = (nat.GpirStageTime * 64)()
    n = ctx.lib.gpir_stage_times(ctx.h, buf, 64)
    out = []
    for e in buf[:max(n, 0)]:
        name = _PHASE_NAMES.get(e.phase, str(e.phase))
        mode = ExecMode.OPERATION_LEVEL.value if e.mode == 0 else ExecMode.STAGE_LEVEL.value
        ws = 0
        if e.phase == 0:
            ws = planner.working_set(Phase.EXPAND_QUERY, e.stage, B, params, config)
        elif e.phase == 3:
            ws = planner.working_set(Phase.COL_TOR, e.stage, B, params, config)
        out.append(StageTiming(name, int(e.stage), int(e.units), mode, ws, e.ms / 1e3,
                               ws if e.mode == 0 else 0))
    return out


def answer_batch(queries, keys_by_client, db, params, hw: HardwareModel | None = None,
                 plan: ExecutionPlan | None = None, mode: ExecMode | None = None, engine: str = "auto",
                 tile=None, pipeline=None, stats: ServeStats | None = None) -> list:
    """Serve a batch end to end on the GPU (src/protocol.py:635-682).

    Every query uses its own client's keys; responses come back in query order
    and are independent of batch composition (bit-identical to the reference)."""
    if not queries:
        return []
    if engine not in _ENGINES:
        raise InvalidArgument(f"unknown row-selection engine {engine!r}")
    if tile is not None or pipeline is not None:
        lay = "p_major" if getattr(getattr(db, "layout", None), "value", "pmajor") in ("pmajor", "p_major") \
            else "transposed"
        b = params.basis
        layout.validate_rowsel(engine, lay, 2 * len(queries), db.config.d1, db.config.d0, b.k, b.n, tile, pipeline)
    for q in queries:
        if q.client_id not in keys_by_client:
            raise InvalidState(f"no uploaded keys for client {q.client_id}")
    ctx = _device_db(db, params).ctx
    qarr = np.empty((len(queries), 2, ctx.k, ctx.n), dtype=np.uint32)
    for i, q in enumerate(queries):
        qarr[i, 0] = q.ct.a.limbs
        qarr[i, 1] = q.ct.b.limbs
    out = answer_raw(qarr, [q.client_id for q in queries], keys_by_client, db, params, hw=hw, plan=plan,
                     mode=mode, engine=engine, stats=stats)
    return [_make_response(q, out[i]) for i, q in enumerate(queries)]


def respond(query, keys, db, params, **kwargs):
    return answer_batch([query], {query.client_id: keys}, db, params, **kwargs)[0]


# north-star aliases
process_batch = answer_batch
process_query = respond
