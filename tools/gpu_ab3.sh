#!/bin/bash
# parity + A/B of alternative libgpir builds (GPIR_LIB) on configs 2 and 3
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_client_gpu.py -x -q -m gpu 2>&1 | tail -1
for cfg in ${CFGS:-2 3}; do
for lib in paper_2604_04696_b200/libgpir.so paper_2604_04696_b200/libgpir_*.so; do
  GPIR_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu --config $cfg --steps 5 --warmup 3 > gpurun_out/ab.log 2>&1
  python - "$lib" "$cfg" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.log").read().strip().splitlines()[-1])
    print("cfg", sys.argv[2], sys.argv[1].split("/")[-1], "QPS", round(d["value"]), {k: round(v, 3) for k, v in d["phases_ms"].items()}, "rs", round(d["roofline"]["frac"], 3))
except Exception as e:
    print(sys.argv[1], "failed", open("gpurun_out/ab.log").read()[-300:])
PY
done
done
