#!/bin/bash
# quick check: full GPU parity suite + one bench line (+ RowSel per-role cycle profile)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_q.log
timeout 300 python bench.py --no-cpu --steps 30 ${BENCH_ARGS} > gpurun_out/bench_q.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]);print(d['value'],d['e2e']['value'],d['phases_ms'],d['roofline']['frac'],d['clocks'])" || tail -5 gpurun_out/bench_q.log
GPIR_TC_PROF=1 timeout 300 python bench.py --no-cpu --steps 3 2>&1 | grep "tc prof" | tail -1
