#!/bin/bash
# GPU test suite (optionally a -k subset) -> gpurun_out/t_gputest.txt
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/t_gputest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/t_gputest.txt
