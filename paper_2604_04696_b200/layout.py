"""RowSel tiling / pipelining configuration objects of the reference's API
(src/layout.py:36, 67-149, 301-307) and their validation.

On the B200 the GEMM tiles and the stream pipelining are fixed by the
tensor-core kernels (csrc/rowsel_tc.cuh), so a caller's TileConfig or
PipelineConfig does not change the schedule; it is still validated exactly
where the reference's engines validate it, so a configuration the reference
rejects raises the same InvalidConfig here (and results never depend on it).
The reference's own config objects are accepted (duck-typed)."""
from __future__ import annotations

from dataclasses import dataclass

from .errors import InvalidArgument, InvalidConfig

DEFAULT_SCRATCH_BYTES = 96 * 1024  # src/layout.py:36


@dataclass(frozen=True)
class TileConfig:
    """Thread-block tile extents; ``bp`` is used by the p-major engine only."""

    bm: int
    bn: int
    bk: int
    bp: int | None = None

    def scratch_bytes(self) -> int:
        return (self.bm * self.bk + self.bn * self.bk) * (self.bp or 1) * 4

    def accumulator_bytes(self) -> int:
        return self.bm * self.bn * (self.bp or 1) * 4

    def validate(self, m: int, n: int, k: int, p: int | None = None,
                 scratch_budget: int = DEFAULT_SCRATCH_BYTES) -> None:
        validate_tile(self, m, n, k, p, scratch_budget)


@dataclass(frozen=True)
class PipelineConfig:
    """Lane/chunk decomposition of the p axis plus the worker pool size."""

    prime_streams: int = 4
    n_chunks: int = 8
    workers: int = 4


def validate_tile(tile, m: int, n: int, k: int, p: int | None, scratch_budget: int) -> None:
    for extent, dim, name in ((tile.bm, m, "bm"), (tile.bn, n, "bn"), (tile.bk, k, "bk")):
        if extent < 1 or dim % extent:
            raise InvalidConfig(f"tile {name}={extent} does not divide problem dim {dim}")
    bp = getattr(tile, "bp", None)
    if bp is not None and (p is None or bp < 1 or p % bp):
        raise InvalidConfig(f"tile bp={bp} does not divide p={p}")
    scratch = (tile.bm * tile.bk + tile.bn * tile.bk) * (bp or 1) * 4
    if scratch > scratch_budget:
        raise InvalidConfig(f"tile scratch {scratch} B exceeds budget {scratch_budget} B")


def validate_rowsel(engine: str, db_layout: str, m: int, d1: int, d0: int, limbs: int, n: int,
                    tile=None, pipeline=None, scratch_budget: int = DEFAULT_SCRATCH_BYTES) -> None:
    """The checks of the reference's row_select_raw for the engine it would
    dispatch (src/protocol.py:448-492, src/layout.py:229-247, 265-277, 351-378)."""
    p = limbs * n
    if engine == "auto":
        engine = "pipeline" if pipeline is not None else ("pmajor" if db_layout == "p_major" else "transposed")
    if engine in ("pmajor",) and tile is not None:
        if getattr(tile, "bp", None) is None:
            raise InvalidConfig("p-major engine requires a bp tile extent")
        validate_tile(tile, m, d1, d0, p, scratch_budget)
    elif engine == "transposed" and tile is not None:
        validate_tile(tile, m, d1, d0, p, scratch_budget)
    elif engine == "pipeline":
        pl = pipeline if pipeline is not None else PipelineConfig()
        if p % limbs:
            raise InvalidArgument(f"p={p} is not a multiple of the limb count {limbs}")
        if pl.prime_streams < 1 or limbs % pl.prime_streams:
            raise InvalidConfig(f"prime_streams={pl.prime_streams} must divide the limb count {limbs}")
        if pl.n_chunks < 1 or n % pl.n_chunks:
            raise InvalidConfig(f"n_chunks={pl.n_chunks} must divide n={n}")
        if tile is not None:  # each (lane, chunk) task runs the transposed engine on its p slice
            p_task = (limbs // pl.prime_streams) * (n // pl.n_chunks)
            validate_tile(tile, m, d1, d0, p_task, scratch_budget)
