#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rowsel or pipeline" > gpurun_out/pytest_rowsel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rowsel.log
tail -2 gpurun_out/pytest_rowsel.log
GPIR_TC_PROF=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu 2>&1 | grep -E "tc prof" | tail -1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
grep -o '"phases_ms.*"total[^}]*}' gpurun_out/bench.log; grep -o '"value": [0-9.]*' gpurun_out/bench.log | head -1
