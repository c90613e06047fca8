#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GPIR_TC_PROF=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --material uniform > gpurun_out/tkp.json 2> gpurun_out/tkp.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --material uniform > gpurun_out/tkb.json 2> gpurun_out/tkb.err
