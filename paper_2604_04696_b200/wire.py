"""Wire format of the server path (mirrors latpir.wire, src/wire.py).

Same framing, codecs, error messages and ParseError offsets as the
reference.  The batch paths are native (libgpir.so `gpir_wire_*`, host code,
no GPU needed): `decode_queries` turns the framed query messages of a whole
batch into ONE contiguous (B, 2, k, n) uint32 array -- pinned when a buffer
from `pinned_queries` is passed, so it feeds `gpir_answer_batch` without a
staging copy -- and `encode_responses` writes the framed response bytes of a
batch in one call.  `load_database` / `save_database` read and write the
reference's GPDB container directly to and from GPU memory.

Single-message helpers (`serialize_query`, `deserialize_response`, ...) are
provided for clients and tests.
"""
from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from . import _native as nat
from .errors import InvalidArgument, ParseError
from .values import BfvCiphertext, ClientQuery, DbConfig, Domain, Response, RnsPoly

MAGIC = b"GPIR"
DB_MAGIC = b"GPDB"
VERSION = 1
_HEADER = struct.Struct("<4sHBQ")
HEADER_BYTES = _HEADER.size  # 15
KIND_PARAMS = 1
KIND_QUERY = 2
KIND_EVKSET = 3
KIND_RESPONSE = 4
KIND_ERROR = 5
KIND_CT = 17
_POLY_ECHO = struct.Struct("<IBB")  # n, k, domain
_ROUTE = struct.Struct("<QI")  # client_id, seq
CT_OVERHEAD = HEADER_BYTES + _POLY_ECHO.size


def serialized_ct_bytes(params) -> int:
    """Exact wire size of one ciphertext message (src/wire.py:48-50)."""
    return CT_OVERHEAD + 2 * params.basis.k * params.n * 4


def _frame(kind: int, payload: bytes) -> bytes:
    return _HEADER.pack(MAGIC, VERSION, kind, len(payload)) + payload


def parse_header(buf: bytes) -> tuple[int, int]:
    """Validate a header; returns (kind, payload length) (src/wire.py:59-69)."""
    lib = nat.load()
    kind, length = C.c_uint32(), C.c_uint64()
    nat.check(lib.gpir_wire_parse_header(C.c_char_p(bytes(buf)), len(buf), C.byref(kind), C.byref(length)))
    return int(kind.value), int(length.value)


def _ct_body(ct) -> bytes:
    n, k = ct.a.limbs.shape[1], ct.a.limbs.shape[0]
    echo = _POLY_ECHO.pack(n, k, 1 if getattr(ct.a, "domain", Domain.NTT).value == "ntt" else 0)
    return echo + np.asarray(ct.a.limbs).astype("<u4").tobytes() + np.asarray(ct.b.limbs).astype("<u4").tobytes()


def serialize_query(q) -> bytes:
    """Framed KIND_QUERY message (src/wire.py:263-264)."""
    return _frame(KIND_QUERY, _ROUTE.pack(q.client_id, q.seq) + _ct_body(q.ct))


def serialize_response(resp) -> bytes:
    """Framed KIND_RESPONSE message (src/wire.py:282-283)."""
    return _frame(KIND_RESPONSE, _ROUTE.pack(resp.client_id, resp.seq) + _ct_body(resp.ct))


def pinned_queries(B: int, k: int, n: int) -> np.ndarray:
    """A page-locked (B, 2, k, n) uint32 buffer for `decode_queries(out=...)`."""
    import torch

    return torch.empty((B, 2, k, n), dtype=torch.int32).pin_memory().numpy().view(np.uint32)


def decode_queries(msgs, n: int, k: int, out: np.ndarray | None = None):
    """Decode a batch of framed query messages in one native call.

    Returns (queries (B, 2, k, n) uint32, client_ids uint64[B], seqs uint32[B]);
    a malformed message raises the reference's ParseError (message, offset) with
    `.index` set to its position in the batch."""
    B = len(msgs)
    if out is None:
        out = np.empty((B, 2, k, n), dtype=np.uint32)
    elif out.shape[0] < B or out.shape[1:] != (2, k, n) or out.dtype != np.uint32 or not out.flags.c_contiguous:
        raise InvalidArgument(f"out must be a contiguous uint32 (>= {B}, 2, {k}, {n}) array")
    out = out[:B]
    bufs = [bytes(m) for m in msgs]
    ptrs = (C.c_void_p * B)(*[C.cast(C.c_char_p(b), C.c_void_p) for b in bufs])
    lens = (C.c_size_t * B)(*[len(b) for b in bufs])
    ids = np.empty(B, dtype=np.uint64)
    seqs = np.empty(B, dtype=np.uint32)
    bad = C.c_uint32(0)
    lib = nat.load()
    try:
        nat.check(lib.gpir_wire_decode_queries(ptrs, lens, B, n, k, nat.ptr(out), ids.ctypes.data_as(
            C.POINTER(C.c_uint64)), nat.ptr(seqs), C.byref(bad)))
    except ParseError as exc:
        exc.index = int(bad.value)
        raise
    return out, ids, seqs


def deserialize_query(buf: bytes, basis) -> ClientQuery:
    """One KIND_QUERY message -> ClientQuery (src/wire.py:267-276)."""
    arr, ids, seqs = decode_queries([buf], basis.n, basis.k)
    return ClientQuery(_ct(arr[0], basis), int(ids[0]), int(seqs[0]))


def _ct(raw, basis) -> BfvCiphertext:
    return BfvCiphertext(RnsPoly(basis, raw[0].astype(np.uint64), Domain.NTT),
                         RnsPoly(basis, raw[1].astype(np.uint64), Domain.NTT))


def response_bytes(n: int, k: int) -> int:
    return int(nat.load().gpir_wire_response_bytes(n, k))


def encode_responses(raw: np.ndarray, client_ids, seqs) -> list[bytes]:
    """(B, 2, k, n) uint32 responses -> framed KIND_RESPONSE messages, one native call."""
    raw = np.ascontiguousarray(raw, dtype=np.uint32)
    B, _, k, n = raw.shape
    ids = np.ascontiguousarray(client_ids, dtype=np.uint64)
    sq = np.ascontiguousarray(seqs, dtype=np.uint32)
    each = response_bytes(n, k)
    buf = np.empty(B * each, dtype=np.uint8)
    nat.check(nat.load().gpir_wire_encode_responses(nat.ptr(raw), ids.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                    nat.ptr(sq), B, n, k, buf.ctypes.data_as(C.c_void_p),
                                                    buf.size))
    mv = buf.tobytes()
    return [mv[i * each:(i + 1) * each] for i in range(B)]


def deserialize_response(buf: bytes, basis) -> Response:
    """KIND_RESPONSE -> Response (src/wire.py:286-294); pure Python (client side)."""
    kind, length = parse_header(buf)
    if len(buf) != HEADER_BYTES + length:
        raise ParseError(f"payload length mismatch: header says {length}, got {len(buf) - HEADER_BYTES}",
                         HEADER_BYTES)
    if kind != KIND_RESPONSE:
        raise ParseError(f"expected response message, got kind {kind}", 6)
    pl = buf[HEADER_BYTES:]
    cid, seq = _ROUTE.unpack_from(pl, 0)
    n, k, _ = _POLY_ECHO.unpack_from(pl, _ROUTE.size)
    if n != basis.n or k != basis.k:
        raise ParseError(f"geometry echo ({n}, {k}) does not match basis ({basis.n}, {basis.k})", _ROUTE.size)
    off = _ROUTE.size + _POLY_ECHO.size
    raw = np.frombuffer(pl, dtype="<u4", count=2 * k * n, offset=off).reshape(2, k, n)
    if off + raw.nbytes != len(pl):
        raise ParseError("trailing bytes after value", off + raw.nbytes)
    return Response(_ct(raw, basis), cid, seq)


class RawKeys:
    """Client key material as the decoded arrays (evks by stage, RGSW(s)); accepted
    wherever ClientKeys is (evk_raw / sk_rgsw_raw)."""

    def __init__(self, n: int, evks: np.ndarray, sk_rgsw: np.ndarray | None):
        self.n = n
        self.evks = evks
        self._rg = sk_rgsw
        self.sk_rgsw = sk_rgsw

    def evk_raw(self, k_aut: int) -> np.ndarray:
        for t in range(self.evks.shape[0]):
            if self.n // (1 << t) + 1 == k_aut:
                return self.evks[t]
        from .errors import InvalidState

        raise InvalidState(f"no evaluation key for automorphism index {k_aut}")

    def sk_rgsw_raw(self) -> np.ndarray:
        if self._rg is None:
            from .errors import InvalidState

            raise InvalidState("this key set has no RGSW of the secret (onion mode needs one)")
        return self._rg


def decode_evkset(buf: bytes, params, stages: int) -> tuple[int, RawKeys]:
    """KIND_EVKSET (src/wire.py:305-318) -> (client_id, RawKeys) holding the
    evaluation keys of the first `stages` expansion stages and RGSW(s)."""
    n, k = params.n, params.basis.k
    ell, zb = params.gadget.ell, params.gadget.z_bits
    evks = np.empty((stages, ell, 2, k, n), dtype=np.uint32)
    rg = np.empty((2 * ell, 2, k, n), dtype=np.uint32)
    cid, has = C.c_uint64(), C.c_int()
    b = bytes(buf)
    nat.check(nat.load().gpir_wire_decode_evkset(C.c_char_p(b), len(b), n, k, zb, ell, stages, nat.ptr(evks),
                                                 nat.ptr(rg), C.byref(cid), C.byref(has)))
    return int(cid.value), RawKeys(n, evks, rg if has.value else None)


def save_database(path: str, db, record_bytes: int | None = None) -> None:
    """Write the GPU-resident DB as a P-major GPDB image (src/wire.py:368-380)."""
    from .protocol import _device_db

    ddb = _device_db(db, db.params)
    rb = db.config.record_bytes if record_bytes is None else record_bytes
    nat.check(ddb.ctx.lib.gpir_db_save(ddb.ctx.h, ddb.handle, path.encode(), rb, db.params.plain_bits), "save")


def load_database(path: str, params, device: int | None = None):
    """Read a GPDB image straight into GPU memory (src/wire.py:383-410); returns
    (EncodedDatabase, params).  Primes (and the plain modulus) are validated
    against `params` with the reference's ParseError."""
    from .protocol import EncodedDatabase, get_context

    ctx = get_context(params, device)
    d0, d1, rb, pb = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
    h = ctx.lib.gpir_db_load(ctx.h, path.encode(), params.plain_bits, C.byref(d0), C.byref(d1), C.byref(rb),
                             C.byref(pb))
    if not h:
        if nat.load().gpir_last_error_offset() >= 0:
            nat.check(-6)
        raise InvalidArgument(nat.last_error())
    cfg = DbConfig(int(d0.value), int(d1.value), int(rb.value))
    return EncodedDatabase(cfg, params, ctx, h), params
