#!/bin/bash
# ExpandQuery operation-level chunking: per-kernel times of the last stage (eq8) for several chunk sizes
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for ch in ${CHUNKS:-0 1024 512 256}; do
  GPIR_OP_CHUNK=$ch GPIR_STAGE_PROF=2 timeout 300 python bench.py --no-cpu --steps 2 --warmup 3 --modes ${PLAN:-ooooooooo/HHHHHo} > gpurun_out/chunk.log 2>&1
  python - "$ch" <<'PY'
import sys, re
lines = [l for l in open("gpurun_out/chunk.log") if l.startswith("[stage prof]")]
# last eq8 block: lines after the last "eq7 " stage line up to the next "eq8 " stage line
i7 = max(i for i, l in enumerate(lines) if re.search(r"\] eq7 ", l))
i8 = min(i for i, l in enumerate(lines) if i > i7 and re.search(r"\] eq8 ", l))
acc = {}
for l in lines[i7 + 1:i8 + 1]:
    parts = l.split()
    name, ms = parts[2], float(parts[-2])
    acc[name] = acc.get(name, 0) + ms
print("chunk", sys.argv[1], {k: round(v, 3) for k, v in acc.items()}, "total", round(sum(acc.values()), 3))
PY
done
