#!/bin/bash
# batch sweep at one DB geometry: QPS, e2e, plan and phases per batch size (BATCHES="1 4 ...", CFG=2)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for b in ${BATCHES:-1 2 4 8 16 32 64 128}; do
  timeout 300 python bench.py --no-cpu --config ${CFG:-2} --batch $b --steps ${STEPS:-10} > gpurun_out/sweep.log 2>&1
  python - "$b" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/sweep.log").read().strip().splitlines()[-1])
    ph = d["phases_ms"]
    print(f"| {sys.argv[1]} | {d['value']:.0f} | {d['e2e']['value']:.0f} | {d['ms_per_step']:.3f} | "
          f"{d['config']['plan_eq']} / {d['config']['plan_ct']} | {ph['ExpandQuery']:.3f} | {ph['RgswAssembly']:.3f} | "
          f"{ph['RowSelPack'] + ph['RowSel']:.3f} | {ph['ColTor']:.3f} | {d['roofline']['frac']:.2f} |")
except Exception as e:
    print(sys.argv[1], "failed", open("gpurun_out/sweep.log").read()[-300:])
PY
done
