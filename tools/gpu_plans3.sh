#!/bin/bash
# plan sweep at config 3 (explicit per-stage modes)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for m in "ooooooooo/HHHHHHHHH" "ooooooooH/HHHHHHHHH" "oooooooHH/HHHHHHHHH" "ooooooHHH/HHHHHHHHH" "ooooooooo/oHHHHHHHH" "ooooooooo/SHHHHHHHH"; do
  timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --material uniform --modes "$m" > "gpurun_out/pl_${m//\//_}.json" 2> "gpurun_out/pl_${m//\//_}.err"
done
