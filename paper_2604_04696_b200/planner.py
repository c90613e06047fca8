"""Hybrid execution planner for the tree phases on B200 (src/planner.py:84-224).

The reference picks operation-level vs stage-fused execution per stage by
comparing the digit-decomposition working set to the last-level cache.  On
B200 the deciding factor is different: the stage-fused kernels run one CTA
per tree node (all limbs and digits of the node stay in shared memory and
registers), so they need enough nodes to fill 148 SMs x 2 resident CTAs;
operation-level kernels expose ELL*K-fold more CTAs per node and win on the
shallow stages.  `build_plan` keeps the reference's API and data types;
`HardwareModel.b200()` carries the B200 constants, and the default rule is
the occupancy rule (`rule="occupancy"`); `rule="working_set"` reproduces the
reference's L2 rule with B200's 126 MB L2.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

from .errors import InvalidArgument


@dataclass(frozen=True)
class HardwareModel:
    """Platform constants.  Defaults are the reference's RTX 5090 model
    (src/planner.py:84-102); use `HardwareModel.b200()` for this GPU."""

    l2_bytes: int = 96 * 1024 * 1024
    dram_bandwidth: float = 1.66e12
    peak_ops: float = 31.5e12
    processors: int = 170
    scratch_bytes: int = 96 * 1024
    resident_ctas: int = 2  # fused-kernel CTAs per SM (96 KiB smem, 128 regs x 256 threads)

    def __post_init__(self):
        for name in ("l2_bytes", "dram_bandwidth", "peak_ops", "processors", "scratch_bytes"):
            if getattr(self, name) <= 0:
                raise InvalidArgument(f"{name} must be positive")

    @classmethod
    def b200(cls) -> "HardwareModel":
        return cls(l2_bytes=126 * 1024 * 1024, dram_bandwidth=6.55e12, peak_ops=36.0e12, processors=148,
                   scratch_bytes=227 * 1024, resident_ctas=2)

    @property
    def ridge_point(self) -> float:
        return self.peak_ops / self.dram_bandwidth


class ExecMode(Enum):
    OPERATION_LEVEL = "op"
    STAGE_LEVEL = "stage"


class Phase(Enum):
    EXPAND_QUERY = "ExpandQuery"
    ROW_SEL = "RowSel"
    COL_TOR = "ColTor"


@dataclass(frozen=True)
class StageProfile:
    phase: Phase
    stage: int
    nodes: int
    footprint_bytes: int
    batch: int
    working_set: int
    mode: ExecMode


@dataclass
class ExecutionPlan:
    expand_stages: list
    coltor_stages: list
    expand_transition: int | None
    coltor_transition: int | None

    def mode_for(self, phase: Phase, stage: int) -> ExecMode:
        stages = self.expand_stages if phase is Phase.EXPAND_QUERY else self.coltor_stages
        return stages[stage].mode

    def rows(self):
        for p in self.expand_stages + self.coltor_stages:
            yield (p.phase.value, p.stage, p.nodes, p.working_set, p.mode.value)

    def to_text(self) -> str:
        lines = ["phase\tstage\tnodes\tworking_set_bytes\tmode"]
        lines += ["\t".join(str(v) for v in r) for r in self.rows()]
        return "\n".join(lines) + "\n"


# tree geometry (src/planner.py:153-173)

def expansion_leaves(d0: int, d1: int, ell: int) -> int:
    return d0 + (d1.bit_length() - 1) * ell


def num_expand_stages(total_leaves: int) -> int:
    return max(math.ceil(math.log2(total_leaves)), 0) if total_leaves > 1 else 0


def expand_nodes(total_leaves: int, stage: int) -> int:
    return min(1 << stage, total_leaves)


def num_coltor_stages(d1: int) -> int:
    return d1.bit_length() - 1


def coltor_nodes(d1: int, stage: int) -> int:
    return d1 >> (stage + 1)


def _poly_bytes(params) -> int:
    return params.basis.k * params.basis.n * 4


def working_set(phase: Phase, stage: int, batch: int, params, config) -> int:
    """Digit-decomposition transient bytes of a stage (src/planner.py:180-191)."""
    ell = params.gadget.ell
    if phase is Phase.EXPAND_QUERY:
        nodes = expand_nodes(expansion_leaves(config.d0, config.d1, ell), stage)
        fp = _poly_bytes(params)
    elif phase is Phase.COL_TOR:
        nodes = coltor_nodes(config.d1, stage)
        fp = 2 * _poly_bytes(params)
    else:
        raise InvalidArgument(f"no working-set model for phase {phase}")
    return nodes * ell * fp * batch


def choose_mode(working_set_bytes: int, hw: HardwareModel) -> ExecMode:
    """Reference L2 rule (src/planner.py:194-196)."""
    return ExecMode.STAGE_LEVEL if working_set_bytes >= hw.l2_bytes else ExecMode.OPERATION_LEVEL


# B200 thresholds of the occupancy rule, measured per stage at config 2
# (profiles/r1_plans.md, r1g_plans.md); identical to kEqStageNodes / kXpStageCts in gpir.cu
EQ_STAGE_NODES = 1 << 62  # r1g: operation-level wins at every ExpandQuery stage (node-batched MAC)
XP_STAGE_CTS = 64


def choose_mode_occupancy(nodes_in_batch: int, hw: HardwareModel, phase: "Phase | None" = None) -> ExecMode:
    """B200 rule: run a stage on the stage-level executor once it has enough
    nodes (ExpandQuery) or ciphertexts (ColTor) to fill the GPU with one CTA
    per node x limb; the operation-level kernels win below that."""
    fill = XP_STAGE_CTS if phase is Phase.COL_TOR else EQ_STAGE_NODES
    return ExecMode.STAGE_LEVEL if nodes_in_batch >= fill else ExecMode.OPERATION_LEVEL


def build_plan(config, params, batch: int, hw: HardwareModel | None = None, rule: str = "occupancy") -> ExecutionPlan:
    """Static per-stage plan for both tree phases (src/planner.py:199-224)."""
    hw = hw or HardwareModel.b200()
    ell = params.gadget.ell
    total = expansion_leaves(config.d0, config.d1, ell)
    expand, coltor = [], []
    et = ct = None
    for t in range(num_expand_stages(total)):
        ws = working_set(Phase.EXPAND_QUERY, t, batch, params, config)
        nodes = expand_nodes(total, t)
        mode = choose_mode(ws, hw) if rule == "working_set" else choose_mode_occupancy(nodes * batch, hw,
                                                                                         Phase.EXPAND_QUERY)
        if mode is ExecMode.STAGE_LEVEL and et is None:
            et = t
        expand.append(StageProfile(Phase.EXPAND_QUERY, t, nodes, _poly_bytes(params), batch, ws, mode))
    saw = False
    for t in range(num_coltor_stages(config.d1)):
        ws = working_set(Phase.COL_TOR, t, batch, params, config)
        nodes = coltor_nodes(config.d1, t)
        mode = choose_mode(ws, hw) if rule == "working_set" else choose_mode_occupancy(nodes * batch, hw,
                                                                                         Phase.COL_TOR)
        if mode is ExecMode.STAGE_LEVEL:
            saw = True
        elif saw and ct is None:
            ct = t
        coltor.append(StageProfile(Phase.COL_TOR, t, nodes, 2 * _poly_bytes(params), batch, ws, mode))
    return ExecutionPlan(expand, coltor, et, ct)


# ---------------------------------------------------------------------------
# analytical model (src/planner.py:227-270)

def rowsel_ops(config, params, batch: int) -> int:
    return params.basis.k * params.basis.n * (2 * batch) * config.d0 * config.d1


def rowsel_bytes(config, params, batch: int) -> int:
    pb = _poly_bytes(params)
    return config.d0 * config.d1 * pb + batch * config.d0 * 2 * pb + batch * config.d1 * 2 * pb


def phase_model(phase: Phase, config, params, batch: int) -> tuple[int, int]:
    ell = params.gadget.ell
    k, n = params.basis.k, params.basis.n
    poly = _poly_bytes(params)
    log_n = n.bit_length() - 1
    if phase is Phase.ROW_SEL:
        return rowsel_ops(config, params, batch), rowsel_bytes(config, params, batch)
    if phase is Phase.EXPAND_QUERY:
        total = expansion_leaves(config.d0, config.d1, ell)
        node_ops = (1 + ell) * (k * n // 2) * log_n + 2 * ell * k * n
        ops = nb = 0
        for t in range(num_expand_stages(total)):
            nodes = expand_nodes(total, t)
            ops += batch * nodes * node_ops
            nb += batch * (nodes * 6 * poly + 2 * ell * poly)
        return ops, nb
    if phase is Phase.COL_TOR:
        node_ops = (2 + 2 * ell) * (k * n // 2) * log_n + 4 * ell * k * n
        ops = nb = 0
        for t in range(num_coltor_stages(config.d1)):
            nodes = coltor_nodes(config.d1, t)
            ops += batch * nodes * node_ops
            nb += batch * (nodes * 6 * poly + 4 * ell * poly)
        return ops, nb
    raise InvalidArgument(f"unknown phase {phase}")


@dataclass(frozen=True)
class RooflineRow:
    phase: str
    ops: int
    bytes: int
    ai: float
    bound: str


@dataclass
class RooflineReport:
    """Arithmetic intensity of each phase against the platform's ridge point
    (src/planner.py:273-302), same fields and text format."""

    hw: HardwareModel
    rows: list

    def to_text(self) -> str:
        out = [f"ridge_point\t{self.hw.ridge_point:.3f}", "phase\tops\tbytes\tai\tbound"]
        out += [f"{r.phase}\t{r.ops}\t{r.bytes}\t{r.ai:.4f}\t{r.bound}" for r in self.rows]
        return "\n".join(out) + "\n"


def roofline_report(hw: HardwareModel, config, params, batch: int) -> RooflineReport:
    """Per-phase ops / bytes from the analytical model (`phase_model`); a phase is
    compute-bound when its intensity reaches hw.ridge_point.  The measured
    counterpart on the B200 is bench.py's phase_roofline / roofline."""
    rows = []
    for ph in (Phase.EXPAND_QUERY, Phase.ROW_SEL, Phase.COL_TOR):
        ops, nb = phase_model(ph, config, params, batch)
        ai = ops / nb
        rows.append(RooflineRow(ph.value, ops, nb, ai, "compute" if ai >= hw.ridge_point else "memory"))
    return RooflineReport(hw, rows)
