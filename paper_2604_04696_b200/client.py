"""Client-side material generated on the GPU (the benchmark
input factory; the reference does this on the CPU, src/he.py:220-271,
423-431, 487-515, src/protocol.py:240-281).

`keygen` samples a client's secret and encrypts its expansion keys and RGSW(s)
straight into a key slot of the context (no host round trip of the ~7 MiB of
key material per client); `queries` encrypts (i*, j*) selections under a
secret.  The RNG is a counter-based hash on the GPU, so samples differ from
numpy's while the distributions and encryption equations are the reference's;
correctness is checked by decrypting the server's responses with the secret
(tests/test_client_gpu.py)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from . import planner


def keygen(ctx, params, slot: int, d0: int, d1: int, seed: int) -> np.ndarray:
    """Install a fresh client's keys for a d0 x d1 DB in key slot `slot`; returns its
    secret's ternary coefficients (int8, n)."""
    stages = planner.num_expand_stages(planner.expansion_leaves(d0, d1, params.gadget.ell))
    secret = np.empty(params.n, dtype=np.int8)
    nat.check(ctx.lib.gpir_client_keygen(ctx.h, slot, stages, seed, params.error_bound,
                                         secret.ctypes.data_as(C.c_void_p)), "client keygen")
    return secret


def queries(ctx, params, secret: np.ndarray, d0: int, d1: int, coords, seed: int) -> np.ndarray:
    """Encrypt the selections `coords` [(i*, j*), ...] under `secret`: (B, 2, k, n) uint32, natural order."""
    ii = np.ascontiguousarray([c[0] for c in coords], dtype=np.uint32)
    jj = np.ascontiguousarray([c[1] for c in coords], dtype=np.uint32)
    out = np.empty((len(coords), 2, params.basis.k, params.n), dtype=np.uint32)
    sc = np.ascontiguousarray(secret, dtype=np.int8)
    nat.check(ctx.lib.gpir_client_queries(ctx.h, sc.ctypes.data_as(C.c_void_p), params.plain_bits,
                                          params.error_bound, d0, d1, nat.ptr(ii), nat.ptr(jj), len(coords), seed,
                                          nat.ptr(out)), "client queries")
    return out
