"""CPU checks of the Python mirror against the reference's own API (latpir from
baseline/_ref, skipped when absent): the analytical phase model and
roofline_report (src/planner.py:246-302), the tile / pipeline validation of
row_select_raw (src/protocol.py:448-492, src/layout.py:67-149, 351-378) and the
comm ledger (src/cluster.py:124-136) give the same numbers and raise the same
errors on the same inputs."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def L():
    if not os.path.isdir(os.path.join(REF, "latpir")):
        pytest.skip("latpir (the reference) is not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import latpir.cluster
    import latpir.he
    import latpir.layout
    import latpir.planner
    import latpir.protocol
    return latpir


@pytest.mark.parametrize("d0,d1,B", [(16, 16, 1), (256, 64, 32), (256, 512, 128), (256, 2048, 256)])
def test_phase_model_and_roofline_report(L, d0, d1, B):
    import paper_2604_04696_b200 as G
    from tests.helpers import to_api
    from oracle import gpir_oracle as O

    P = L.he.default_params()
    p = to_api(O.default_params())
    cfg_r, cfg = L.protocol.DbConfig(d0, d1, 1024), G.DbConfig(d0, d1, 1024)
    for ph_r, ph in ((L.planner.Phase.EXPAND_QUERY, G.Phase.EXPAND_QUERY), (L.planner.Phase.ROW_SEL, G.Phase.ROW_SEL),
                     (L.planner.Phase.COL_TOR, G.Phase.COL_TOR)):
        assert L.planner._phase_model(ph_r, cfg_r, P, B) == G.planner.phase_model(ph, cfg, p, B)
    hw_r = L.planner.HardwareModel()
    hw = G.HardwareModel()
    want = L.planner.roofline_report(hw_r, cfg_r, P, B).to_text()
    assert G.planner.roofline_report(hw, cfg, p, B).to_text() == want


def test_tile_and_pipeline_validation(L):
    from paper_2604_04696_b200 import errors, layout

    TC, PC = L.layout.TileConfig, L.layout.PipelineConfig
    k, n = 4, 4096
    cases = [("auto", "p_major", TC(3, 8, 8, bp=1), None), ("auto", "p_major", TC(2, 8, 8), None),
             ("auto", "p_major", TC(2, 8, 8, bp=4), None), ("auto", "p_major", TC(2, 8, 8, bp=3), None),
             ("auto", "p_major", TC(64, 64, 64, bp=32), None), ("transposed", "p_major", TC(2, 7, 8), None),
             ("auto", "p_major", None, PC(prime_streams=3)), ("auto", "p_major", None, PC(n_chunks=6)),
             ("auto", "p_major", TC(2, 8, 8, bp=4), PC(prime_streams=2, n_chunks=4)),
             ("auto", "transposed", TC(2, 16, 16), None)]
    for engine, lay, tile, pl in cases:
        ref_err = None
        try:  # the reference's own checks, as row_select_raw / its engines run them
            m, d1, d0, p = 2, 8, 8, k * n
            eng = engine if engine != "auto" else ("pipeline" if pl is not None else
                                                    ("pmajor" if lay == "p_major" else "transposed"))
            if eng == "pmajor" and tile is not None:
                if tile.bp is None:
                    raise L.errors.InvalidConfig("p-major engine requires a bp tile extent")
                tile.validate(m, d1, d0, p)
            elif eng == "transposed" and tile is not None:
                tile.validate(m, d1, d0, p)
            elif eng == "pipeline":
                if k % pl.prime_streams:
                    raise L.errors.InvalidConfig("prime_streams")
                if n % pl.n_chunks:
                    raise L.errors.InvalidConfig("n_chunks")
                if tile is not None:
                    tile.validate(m, d1, d0, (k // pl.prime_streams) * (n // pl.n_chunks))
        except L.errors.InvalidConfig as e:
            ref_err = e
        if ref_err is None:
            layout.validate_rowsel(engine, lay, 2, 8, 8, k, n, tile, pl)
        else:
            with pytest.raises(errors.InvalidConfig):
                layout.validate_rowsel(engine, lay, 2, 8, 8, k, n, tile, pl)


def test_comm_ledger_matches_reference(L):
    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200.cluster import Strategy, comm_bytes

    P = L.he.default_params()
    for d0, d1, B, nw in ((256, 64, 32, 2), (256, 512, 128, 8), (16, 16, 4, 4)):
        cfg_r = L.protocol.DbConfig(d0, d1, 1024)
        cfg = G.DbConfig(d0, d1, 1024)
        for sr, s in ((L.cluster.Strategy.SHARD_ALL_GATHER, Strategy.SHARD_ALL_GATHER),
                      (L.cluster.Strategy.SHARD_AGGREGATE, Strategy.SHARD_AGGREGATE),
                      (L.cluster.Strategy.NAIVE_BATCH, Strategy.NAIVE_BATCH)):
            a = L.cluster.comm_bytes(sr, cfg_r, B, nw, P)
            b = comm_bytes(s, cfg, B, nw, G.default_params())
            assert (a.after_expand_bytes, a.after_coltor_bytes, a.rgsw_sidecar_bytes) == \
                (b.after_expand_bytes, b.after_coltor_bytes, b.rgsw_sidecar_bytes)
