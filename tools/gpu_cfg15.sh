#!/bin/bash
# configs 1 and 5 bench lines + reference arm at configs 1, 2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python bench.py --config 1 > gpurun_out/c1.json 2> gpurun_out/c1.err
timeout 1500 python bench.py --config 5 --no-cpu --steps 3 > gpurun_out/c5.json 2> gpurun_out/c5.err
timeout 600 python bench.py --impl reference --config 1 --steps 3 --warmup 1 > gpurun_out/r1.json 2> gpurun_out/r1.err
timeout 900 python bench.py --impl reference --config 2 --steps 5 --warmup 1 > gpurun_out/r2.json 2> gpurun_out/r2.err
timeout 900 python bench.py --impl reference --config 4 --steps 2 --warmup 0 > gpurun_out/r4.json 2> gpurun_out/r4.err
