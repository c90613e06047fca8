#!/bin/bash
# quick A/B: parity subset + configs 3 and 2 (uniform material)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "${PYTEST_K:-expand_stages or subs or pipeline or config or interleaved}" > gpurun_out/ab_test.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/ab_test.txt
for cfg in 3 2; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --material uniform > gpurun_out/ab_$cfg.json 2> gpurun_out/ab_$cfg.err
done
