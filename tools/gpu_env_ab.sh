#!/bin/bash
# A/B one environment knob on one bench config: VAR=GPIR_TC_RA VALS="0 64" CFG=3 bash tools/gpu_env_ab.sh
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in ${VALS}; do
  env ${VAR}=$v timeout 300 python bench.py --no-cpu --config ${CFG:-2} --steps ${STEPS:-5} --warmup 3 > gpurun_out/ab.log 2>&1
  python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.log").read().strip().splitlines()[-1])
print(sys.argv[1], "QPS", round(d["value"]), {k: round(v, 3) for k, v in d["phases_ms"].items()})
PY
done
