#!/bin/bash
# round 2: benches after the stats / layout changes (configs 3, 2, 4) + the ncu evidence of configs 3 and 2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu > gpurun_out/g_b3.json 2> gpurun_out/g_b3.err
timeout 600 python bench.py --config 2 --no-cpu > gpurun_out/g_b2.json 2> gpurun_out/g_b2.err
timeout 900 python bench.py --config 4 --no-cpu --steps 5 > gpurun_out/g_b4.json 2> gpurun_out/g_b4.err
bash tools/gpu_prof_r2.sh > gpurun_out/g_prof.log 2>&1
