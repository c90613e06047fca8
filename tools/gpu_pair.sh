#!/bin/bash
# k_rowsel_tk dedicated A slots (GPIR_TK_ARING=1): parity + config 3 timing both ways
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GPIR_TK_ARING=1 timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rowsel or config or interleaved or capacity or alternating" > gpurun_out/pr_test.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pr_test.txt
for e in 0 1; do
  GPIR_TK_ARING=$e timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu --material uniform > gpurun_out/pr_$e.json 2> gpurun_out/pr_$e.err
  GPIR_TK_ARING=$e GPIR_TC_PROF=1 timeout 300 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu --material uniform > gpurun_out/pr_p$e.json 2> gpurun_out/pr_p$e.err
done
