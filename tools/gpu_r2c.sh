#!/bin/bash
# round 2: k_rowsel_tk timing probes at config 3 (GPIR_TK_Y: 1 Y-layout writes, 2 no writes, 3 no math)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu --material uniform --config 3"
for env in "GPIR_TK_Y=1" "GPIR_TK_Y=2" "GPIR_TK_Y=3" "GPIR_TK_Y=1 GPIR_TC_PROF=1" "GPIR_TK_Y=3 GPIR_TC_PROF=1"; do
  env $env timeout 600 $B > "gpurun_out/c_${env// /_}.json" 2> "gpurun_out/c_${env// /_}.err"
done
