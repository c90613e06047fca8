#!/bin/bash
# ColTor stage 0: stage-level H vs split S, alternated, config 3 (3 rounds x 2 plans, 20 steps)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for r in 1 2 3; do
  for m in "ooooooooo/HHHHHHHHH" "ooooooooo/SHHHHHHHH" "ooooooooo/SSHHHHHHH"; do
    timeout 600 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu --material uniform --modes "$m" > "gpurun_out/s0_${r}_${m//\//_}.json" 2>/dev/null
  done
done
