#!/bin/bash
# round 2: grouped-diagonal k_rowsel_tk + Y transpose: parity subset, config 3/2 timing, tk profile counters
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/d_gputest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/d_gputest.txt
B="python bench.py --steps 5 --warmup 3 --no-cpu --material uniform"
timeout 600 $B --config 3 > gpurun_out/d_b3.json 2> gpurun_out/d_b3.err
GPIR_TC_PROF=1 timeout 600 $B --config 3 --steps 1 > gpurun_out/d_b3p.json 2> gpurun_out/d_b3p.err
timeout 600 $B --config 2 > gpurun_out/d_b2.json 2> gpurun_out/d_b2.err
