#!/bin/bash
# round 2 check: build freshness, GPU tests, a config-3 bench with stage timing
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
( nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; free -g; nproc ) > gpurun_out/env.txt 2>&1
python -c "from paper_2604_04696_b200 import build as b; print(b.build())" > gpurun_out/build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gputest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.txt
GPIR_STAGE_PROF=2 timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/b3.json 2> gpurun_out/b3.err
echo "bench3 rc=$?" >> gpurun_out/b3.err
GPIR_STAGE_PROF=2 timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/b2.json 2> gpurun_out/b2.err
tail -5 gpurun_out/gputest.txt
