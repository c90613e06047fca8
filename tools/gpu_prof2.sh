#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu"
for k in ${KERNELS:-k_eq_fused}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-3} -c 1 -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
