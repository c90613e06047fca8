#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for e in 0 1; do
GPIR_TK_PAIR=$e GPIR_TC_PROF=1 timeout 300 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu --material uniform > gpurun_out/pr_p$e.json 2> gpurun_out/pr_p$e.err
done
