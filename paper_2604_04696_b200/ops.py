"""Operator-level entry points on the GPU, with the reference's array
signatures — used by the parity tests to pin each kernel separately.

  ntt_raw / intt_raw          src/ring.py:408-453
  digits (DigitExtractor)     src/he.py:323-367
  expand_stage                src/planner.py:321-381
  external_product_batch      src/planner.py:384-435
  coltor_stage                src/planner.py:438-463
  row_select                  src/protocol.py:448-501 (P-major GEMM engine)
"""
from __future__ import annotations

import numpy as np

from . import _native as nat
from .errors import InvalidArgument
from .protocol import EncodedDatabase, _device_db, get_context
from .values import U64


class _P:  # minimal params shim from (basis, gadget)
    def __init__(self, basis, gadget):
        self.basis, self.gadget = basis, gadget


def _ctx(basis, gadget=None):
    from .values import GadgetConfig

    if gadget is None:  # the NTT does not depend on the gadget; pick a compiled one
        g = {4: GadgetConfig(22, 5), 2: GadgetConfig(11, 5)}.get(basis.k, GadgetConfig(22, 5))
        if basis.n == 64:
            g = GadgetConfig(7, 6)
        gadget = g
    return get_context(_P(basis, gadget))


def _u32(a):
    return np.ascontiguousarray(np.asarray(a), dtype=np.uint32)


def _mode(mode) -> int:
    """ExecMode / 'op' / 'stage' / 'split' / 'hybrid' -> C-ABI mode code (include/gpir.h)."""
    v = getattr(mode, "value", mode)
    return {"op": 0, 0: 0, "stage": 1, 1: 1, "split": 2, 2: 2, "hybrid": 3, 3: 3}[v]


def ntt_raw(x, basis, gadget=None):
    x = np.asarray(x)
    ctx = _ctx(basis, gadget)
    xi = _u32(x).reshape(-1, basis.k, basis.n)
    out = np.empty_like(xi)
    nat.check(ctx.lib.gpir_op_ntt(ctx.h, nat.ptr(xi), nat.ptr(out), xi.shape[0], 0), "ntt")
    return out.reshape(x.shape).astype(U64)


def intt_raw(x, basis, gadget=None):
    x = np.asarray(x)
    ctx = _ctx(basis, gadget)
    xi = _u32(x).reshape(-1, basis.k, basis.n)
    out = np.empty_like(xi)
    nat.check(ctx.lib.gpir_op_ntt(ctx.h, nat.ptr(xi), nat.ptr(out), xi.shape[0], 1), "intt")
    return out.reshape(x.shape).astype(U64)


def digits(coeff, basis, gadget):
    """Signed gadget digits of coefficient-domain limbs (..., k, n) -> (..., ell, n) int64."""
    coeff = np.asarray(coeff)
    ctx = _ctx(basis, gadget)
    ci = _u32(coeff).reshape(-1, basis.k, basis.n)
    out = np.empty((ci.shape[0], gadget.ell, basis.n), dtype=np.int32)
    nat.check(ctx.lib.gpir_op_digits(ctx.h, nat.ptr(ci), nat.ptr(out, nat.C.c_int32), ci.shape[0]), "digits")
    return out.reshape(coeff.shape[:-2] + (gadget.ell, basis.n)).astype(np.int64)


def expand_stage(state, ksks, k_aut, mono_neg, basis, gadget, mode, arena=None):
    """One ExpandQuery stage: (B, C, 2, k, n) -> (B, 2C, 2, k, n) (mono_neg is implied by k_aut)."""
    state = _u32(state)
    ksks = _u32(ksks)
    B, C = state.shape[:2]
    t = (basis.n // (int(k_aut) - 1)).bit_length() - 1
    if basis.n // (1 << t) + 1 != int(k_aut):
        raise InvalidArgument(f"k_aut={k_aut} is not an expansion-stage index n/2^t + 1")
    ctx = _ctx(basis, gadget)
    out = np.empty((B, 2 * C) + state.shape[2:], dtype=np.uint32)
    nat.check(ctx.lib.gpir_op_expand_stage(ctx.h, nat.ptr(state), B, C, nat.ptr(ksks), t, _mode(mode), nat.ptr(out)),
              "expand_stage")
    return out.astype(U64)


def external_product_batch(cts, rgsw_rows, basis, gadget, mode, arena=None):
    cts = _u32(cts)
    rows = _u32(rgsw_rows)
    B, M = cts.shape[:2]
    ctx = _ctx(basis, gadget)
    out = np.empty_like(cts)
    nat.check(ctx.lib.gpir_op_ext_product(ctx.h, nat.ptr(cts), B, M, nat.ptr(rows), _mode(mode), nat.ptr(out)),
              "external_product")
    return out.astype(U64)


def coltor_stage(state, rgsw_rows, basis, gadget, mode, arena=None):
    state = _u32(state)
    rows = _u32(rgsw_rows)
    B, C = state.shape[:2]
    if C % 2:
        raise InvalidArgument("tournament stage needs an even number of ciphertexts")
    ctx = _ctx(basis, gadget)
    out = np.empty((B, C // 2) + state.shape[2:], dtype=np.uint32)
    nat.check(ctx.lib.gpir_op_coltor_stage(ctx.h, nat.ptr(state), B, C, nat.ptr(rows), _mode(mode), nat.ptr(out)),
              "coltor_stage")
    return out.astype(U64)


_ENGINE_CODES = {"auto": 0, "cudacore": 1, "tensorcore": 2}


def row_select(row_cts, db, params, engine: str = "auto"):
    """row_cts (B, d0, 2, k, n) -> selected (B, d1, 2, k, n) on the GPU.

    engine: "auto" (tensor cores when the shape allows), "cudacore", "tensorcore"."""
    ddb = _device_db(db, params)
    nat.check(ddb.ctx.lib.gpir_set_rowsel_engine(ddb.ctx.h, _ENGINE_CODES[engine]), "rowsel engine")
    rc = _u32(row_cts)
    B = rc.shape[0]
    if rc.shape[1] != ddb.config.d0:
        raise InvalidArgument(f"expanded row count {rc.shape[1]} != database d0 {ddb.config.d0}")
    out = np.empty((B, ddb.config.d1) + rc.shape[2:], dtype=np.uint32)
    try:
        nat.check(ddb.ctx.lib.gpir_op_rowsel(ddb.ctx.h, nat.ptr(rc), B, ddb.handle, nat.ptr(out)), "rowsel")
    finally:
        ddb.ctx.lib.gpir_set_rowsel_engine(ddb.ctx.h, 0)
    return out.astype(U64)
