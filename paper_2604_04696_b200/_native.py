"""ctypes binding of libgpir.so (include/gpir.h).

The shared library is built in-tree (`python -m paper_2604_04696_b200.build` or
`__graft_entry__.build()`).  There is no CPU fallback: if the library or a GPU
is missing, every entry point raises `NativeError`.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import InvalidArgument, InvalidConfig, InvalidState, NativeError, ParseError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GPIR_LIB", os.path.join(HERE, "libgpir.so"))

_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)


class GpirStats(C.Structure):
    _fields_ = [
        ("ms_expand", C.c_float), ("ms_rgsw", C.c_float), ("ms_rowsel", C.c_float),
        ("ms_coltor", C.c_float), ("ms_total", C.c_float), ("ms_h2d", C.c_float),
        ("ms_d2h", C.c_float), ("launches", C.c_uint32), ("ms_rowsel_kernel", C.c_float),
        ("ms_rowsel_transpose", C.c_float),
    ]


class GpirStageTime(C.Structure):
    _fields_ = [("phase", C.c_uint8), ("mode", C.c_uint8), ("stage", C.c_uint16), ("units", C.c_uint32),
                ("ms", C.c_float)]


# name -> (restype, argtypes)
_SIGS = {
    "gpir_last_error": (C.c_char_p, []),
    "gpir_version": (C.c_char_p, []),
    "gpir_supported": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32]),
    "gpir_ctx_create": (C.c_void_p, [C.c_int, C.c_uint32, C.c_uint32, _u32p, _u32p, C.c_uint32, C.c_uint32]),
    "gpir_ctx_destroy": (None, [C.c_void_p]),
    "gpir_ctx_device": (C.c_int, [C.c_void_p]),
    "gpir_set_rowsel_engine": (C.c_int, [C.c_void_p, C.c_int]),
    "gpir_set_graphs": (C.c_int, [C.c_void_p, C.c_int]),
    "gpir_set_capacity": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32]),
    "gpir_launch_count": (C.c_uint64, []),
    "gpir_db_encode": (C.c_void_p, [C.c_void_p, _u8p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
    "gpir_db_upload": (C.c_void_p, [C.c_void_p, _u32p, C.c_uint32, C.c_uint32]),
    "gpir_db_encode_dev": (C.c_void_p, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
    "gpir_db_compact": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gpir_db_download": (C.c_int, [C.c_void_p, C.c_void_p, _u32p]),
    "gpir_db_destroy": (None, [C.c_void_p, C.c_void_p]),
    "gpir_db_bytes": (C.c_size_t, [C.c_void_p]),
    "gpir_keys_put": (C.c_int, [C.c_void_p, C.c_int, _u32p, C.c_uint32, _u32p]),
    "gpir_keys_drop": (C.c_int, [C.c_void_p, C.c_int]),
    "gpir_answer_batch": (C.c_int, [C.c_void_p, C.c_void_p, _u32p, _i32p, C.c_uint32, _u8p, C.c_uint32, _u8p,
                                    C.c_uint32, _u32p, C.POINTER(GpirStats)]),
    "gpir_answer_batch_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, _i32p, C.c_uint32, _u8p, C.c_uint32,
                                        _u8p, C.c_uint32, C.c_void_p, C.c_void_p, C.POINTER(GpirStats)]),
    "gpir_plan": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, _u8p, C.c_uint32, _u8p, C.c_uint32]),
    "gpir_shard_answer": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, _i32p, C.c_uint32, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.POINTER(GpirStats)]),
    "gpir_coltor_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                  C.c_void_p]),
    "gpir_sharded_expand": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, _i32p, C.c_uint32, C.c_void_p,
                                      C.c_void_p]),
    "gpir_sharded_rowsel": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
    "gpir_sharded_rowsel_coltor": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p,
                                             C.c_void_p]),
    "gpir_sharded_coltor": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
    "gpir_sharded_rgsw": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]),
    "gpir_layout_convert": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "gpir_last_error_offset": (C.c_int64, []),
    "gpir_set_stage_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "gpir_client_keygen": (C.c_int, [C.c_void_p, C.c_int, C.c_uint32, C.c_uint64, C.c_uint32, C.c_void_p]),
    "gpir_client_queries": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, _u32p,
                                      _u32p, C.c_uint32, C.c_uint64, _u32p]),
    "gpir_stage_times": (C.c_int, [C.c_void_p, C.POINTER(GpirStageTime), C.c_uint32]),
    "gpir_db_load": (C.c_void_p, [C.c_void_p, C.c_char_p, C.c_uint32, _u32p, _u32p, _u32p, _u32p]),
    "gpir_db_save": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_uint32, C.c_uint32]),
    "gpir_wire_parse_header": (C.c_int, [C.c_void_p, C.c_size_t, _u32p, C.POINTER(C.c_uint64)]),
    "gpir_wire_decode_queries": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_uint32, C.c_uint32,
                                           C.c_uint32, _u32p, C.POINTER(C.c_uint64), _u32p, _u32p]),
    "gpir_wire_response_bytes": (C.c_size_t, [C.c_uint32, C.c_uint32]),
    "gpir_wire_encode_responses": (C.c_int, [_u32p, C.POINTER(C.c_uint64), _u32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                             C.c_void_p, C.c_size_t]),
    "gpir_wire_decode_evkset": (C.c_int, [C.c_void_p, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, _u32p, _u32p, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]),
    "gpir_op_ntt": (C.c_int, [C.c_void_p, _u32p, _u32p, C.c_uint32, C.c_int]),
    "gpir_op_digits": (C.c_int, [C.c_void_p, _u32p, _i32p, C.c_uint32]),
    "gpir_op_expand_stage": (C.c_int, [C.c_void_p, _u32p, C.c_uint32, C.c_uint32, _u32p, C.c_uint32, C.c_int, _u32p]),
    "gpir_op_ext_product": (C.c_int, [C.c_void_p, _u32p, C.c_uint32, C.c_uint32, _u32p, C.c_int, _u32p]),
    "gpir_op_coltor_stage": (C.c_int, [C.c_void_p, _u32p, C.c_uint32, C.c_uint32, _u32p, C.c_int, _u32p]),
    "gpir_op_rowsel": (C.c_int, [C.c_void_p, _u32p, C.c_uint32, C.c_void_p, _u32p]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load(path: str | None = None):
    """Load (once) and return the ctypes library; raises NativeError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise NativeError(f"libgpir.so not built at {p}; run __graft_entry__.build()")
        try:
            lib = C.CDLL(p)
        except OSError as exc:
            raise NativeError(f"cannot load {p}: {exc}") from None
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().gpir_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == -1:
        raise InvalidArgument(msg)
    if rc == -2:
        raise InvalidState(msg)
    if rc == -3:
        raise InvalidConfig(msg)
    if rc == -6:  # the reference's message and byte offset, unprefixed
        raise ParseError(last_error(), int(load().gpir_last_error_offset()))
    raise NativeError(f"{msg} (status {rc})")


def ptr(a, ctype=C.c_uint32):
    """ctypes pointer to a C-contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))
