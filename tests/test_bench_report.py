"""server.run_bench: the reference's BenchReport formats (src/server.py:371-455)
filled with per-stage GPU timings (gpir_stage_times)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_run_bench_report():
    import paper_2604_04696_b200 as G
    from paper_2604_04696_b200 import server

    p = G.HeParams(G.default_basis(4096), 16)
    d0, d1, rb = 16, 8, 1024
    rng = np.random.default_rng(5)
    recs = rng.integers(0, 256, size=(d0 * d1, rb), dtype=np.uint8)
    db = G.encode_database_array(recs, G.DbConfig(d0, d1, rb), p)
    rep = server.run_bench(db, p, batches=2, batch=4)
    assert rep.batch == 4 and rep.batches == 2 and rep.qps > 0
    assert set(rep.phase_ms_per_query) == {"ExpandQuery", "RgswAssembly", "RowSel", "ColTor"}
    assert all(v > 0 for v in rep.phase_ms_per_query.values())
    phases = {r[0] for r in rep.stage_rows}
    assert phases == {"ExpandQuery", "RgswAssembly", "ColTor"}
    eq = sorted(r[1] for r in rep.stage_rows if r[0] == "ExpandQuery")
    total = G.planner.expansion_leaves(d0, d1, p.gadget.ell)
    assert eq == list(range(G.planner.num_expand_stages(total)))
    assert rep.stage_csv().startswith("phase,stage,nodes,working_set_bytes,mode,amortized_ms\n")
    text = rep.to_text()
    assert "qps\t" in text and "amortized_ms\tExpandQuery\t" in text and "-- plan --" in text
