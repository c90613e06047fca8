#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "rowsel or pipeline" > gpurun_out/pytest_pst.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pst.log
for p in 8 4 2; do
  GPIR_TC_PST=$p timeout 300 python bench.py --no-cpu --steps 30 > gpurun_out/bench_pst$p.log 2>&1
  echo "PST=$p"; python -c "
import json;d=json.loads(open('gpurun_out/bench_pst$p.log').read().strip().splitlines()[-1]);print(d['value'],d['phases_ms'],d['roofline']['frac'],d['clocks'])"
done
GPIR_TC_PROF=1 timeout 300 python bench.py --no-cpu --steps 3 2>&1 | grep "tc prof" | tail -2
