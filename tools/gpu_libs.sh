#!/bin/bash
# compare per-stage times across alternative libgpir builds (GPIR_LIB)
cd "$GRAFT_REPO_ROOT" || exit 1
for lib in paper_2604_04696_b200/libgpir.so paper_2604_04696_b200/libgpir_*.so; do
  echo "=== $lib"
  GPIR_LIB=$PWD/$lib GPIR_STAGE_PROF=1 timeout 300 python bench.py --no-cpu --steps 3 ${BENCH_ARGS} > gpurun_out/lib.log 2>&1
  grep "stage prof" gpurun_out/lib.log | tail -18 | awk '{printf "%s %s %s | ", $3, $4, $5} END {print ""}'
  python -c "
import json;d=json.loads(open('gpurun_out/lib.log').read().strip().splitlines()[-1]);print('QPS',round(d['value']),d['phases_ms'])" 2>/dev/null || tail -3 gpurun_out/lib.log
done
