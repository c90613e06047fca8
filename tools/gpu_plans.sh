#!/bin/bash
# per-stage device times (GPIR_STAGE_PROF) for several ExpandQuery/ColTor plans at config 2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for plan in "" "FFFFFFFFF/FFFFFF" "ooooooooo/oooooo" "SSSSSSSSS/SSSSSS" ${PLANS}; do
  echo "=== plan '${plan}'"
  GPIR_STAGE_PROF=1 timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 ${plan:+--modes $plan} ${BENCH_ARGS} > gpurun_out/plan.log 2>&1
  grep "stage prof" gpurun_out/plan.log | tail -18 | awk '{printf "%s %s %s | ", $3, $4, $5} END {print ""}'
  python -c "
import json;d=json.loads(open('gpurun_out/plan.log').read().strip().splitlines()[-1]);print('QPS',round(d['value']),d['phases_ms'])" 2>/dev/null || tail -3 gpurun_out/plan.log
done
