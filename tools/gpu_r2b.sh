#!/bin/bash
# round 2: A/B of the RowSel kernels and the fused A operand at configs 2/3, ncu of the RowSel kernels
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu"
for cfg in 3 2; do
  for env in "GPIR_TK=1" "GPIR_TK=0" "GPIR_TK=0 GPIR_FUSE_A8=0"; do
    env $env timeout 600 $B --config $cfg > gpurun_out/ab_${cfg}_${env// /_}.json 2> gpurun_out/ab_${cfg}_${env// /_}.err
  done
done
P="python bench.py --steps 1 --warmup 3 --no-cpu --config 3"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rowsel_tk -s 2 -c 1 -o gpurun_out/r2_tk3 $P > gpurun_out/ncu_tk3.log 2>&1
GPIR_TK=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rowsel_tc -s 2 -c 1 -o gpurun_out/r2_tc3 $P > gpurun_out/ncu_tc3.log 2>&1
ls gpurun_out
