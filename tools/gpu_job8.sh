#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench2.log 2>&1; grep -o '"value": [0-9.]*' gpurun_out/bench2.log | head -1; grep -o '"phases_ms[^}]*}' gpurun_out/bench2.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --config 3 > gpurun_out/bench3.log 2>&1; grep -o '"value": [0-9.]*' gpurun_out/bench3.log | head -1; grep -o '"phases_ms[^}]*}' gpurun_out/bench3.log; tail -2 gpurun_out/bench3.log | cut -c1-300
