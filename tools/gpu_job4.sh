#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rowsel" > gpurun_out/pytest_rowsel.log 2>&1; echo "rowsel rc=$?" >> gpurun_out/pytest_rowsel.log
tail -15 gpurun_out/pytest_rowsel.log
if grep -q "rowsel rc=0" gpurun_out/pytest_rowsel.log; then
  timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
  tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log
fi
