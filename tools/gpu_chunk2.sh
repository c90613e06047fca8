#!/bin/bash
# op-level chunk budget A/B at config 3
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for b in 2 4 8 16; do
  GPIR_OP_BUDGET_GIB=$b timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu --material uniform > gpurun_out/ch_$b.json 2> gpurun_out/ch_$b.err
done
