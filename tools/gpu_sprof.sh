#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GPIR_STAGE_PROF=2 timeout 600 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu --material uniform > gpurun_out/sp3.json 2> gpurun_out/sp3.err
