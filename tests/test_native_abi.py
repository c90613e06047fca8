"""CPU-side checks of the C ABI: the library loads and exports every symbol
declared in include/gpir.h; host-side API logic that needs no GPU."""
import os
import re

import pytest

from tests.conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "gpir.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gpir_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_boundary():
    names = _declared()
    for must in ("gpir_ctx_create", "gpir_db_encode", "gpir_keys_put", "gpir_answer_batch", "gpir_answer_batch_dev",
                 "gpir_op_ntt", "gpir_op_rowsel", "gpir_shard_answer", "gpir_coltor_dev"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2604_04696_b200 import _native

    lib = _native.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_native.EXPORTED)


def test_supported_combinations():
    from paper_2604_04696_b200 import _native

    lib = _native.load()
    assert lib.gpir_supported(4096, 4, 5) == 1
    assert lib.gpir_supported(256, 2, 5) == 1
    assert lib.gpir_supported(64, 2, 6) == 1
    assert lib.gpir_supported(4096, 3, 5) == 0
    assert lib.gpir_supported(1000, 4, 5) == 0


def test_ctx_create_rejects_unsupported():
    import numpy as np

    from paper_2604_04696_b200 import _native

    lib = _native.load()
    q = np.array([97, 193], dtype=np.uint32)
    h = lib.gpir_ctx_create(0, 1000, 2, _native.ptr(q), _native.ptr(q), 11, 5)
    assert not h
    assert "unsupported" in _native.last_error()


def test_error_mapping():
    from paper_2604_04696_b200 import InvalidArgument, InvalidConfig, InvalidState, NativeError, _native

    for rc, cls in ((-1, InvalidArgument), (-2, InvalidState), (-3, InvalidConfig), (-4, NativeError)):
        with pytest.raises(cls):
            _native.check(rc, "x")


def test_params_match_reference_profiles(golden):
    import paper_2604_04696_b200 as G

    _, vec = golden
    p = G.default_params()
    assert [m.q for m in p.basis.moduli] == [int(v) for v in vec["prod_qs"]]
    assert [m.two_n_root for m in p.basis.moduli] == [int(v) for v in vec["prod_psis"]]
    t = G.test_params()
    assert [m.q for m in t.basis.moduli] == [int(v) for v in vec["proto_qs"]]
    assert t.gadget.ell == 5


def test_planner_laws():
    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200 import planner

    p = G.default_params()
    hw = G.HardwareModel()
    # the reference's working-set spike (tests/test_planner.py:38-43)
    ws = planner.working_set(G.Phase.COL_TOR, 0, 32, p, G.DbConfig(256, 512, 16384))
    assert ws == 5_368_709_120
    plan = G.build_plan(G.DbConfig(256, 64, 8192), p, 32, G.HardwareModel.b200())
    modes = "".join("F" if s.mode is G.ExecMode.STAGE_LEVEL else "o" for s in plan.expand_stages)
    assert modes == "ooooooooo"   # r1g: operation-level at every ExpandQuery stage (profiles/r1g_plans.md)
    cmodes = "".join("F" if s.mode is G.ExecMode.STAGE_LEVEL else "o" for s in plan.coltor_stages)
    assert cmodes == "FFFFFo"     # ColTor: stage-level while B * pairs >= 64, then operation-level (r1g_plans.md)
    ref_rule = G.build_plan(G.DbConfig(16, 16, 16384), p, 1, hw, rule="working_set")
    assert all(s.mode is G.ExecMode.OPERATION_LEVEL for s in ref_rule.expand_stages + ref_rule.coltor_stages)


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2604_04696_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "oracle" not in re.sub(r"#.*|\"\"\"[\s\S]*?\"\"\"", "", src), f
