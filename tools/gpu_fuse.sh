#!/bin/bash
# A/B of the A-operand pack fused into the last ExpandQuery stage (GPIR_FUSE_A8=1) + its parity
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GPIR_FUSE_A8=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "config or interleaved or capacity or pipeline or graph or dropin" > gpurun_out/fu_test.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/fu_test.txt
for cfg in 3 2; do
  for f in 0 1; do
    GPIR_FUSE_A8=$f timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --material uniform > gpurun_out/fu_${cfg}_$f.json 2> gpurun_out/fu_${cfg}_$f.err
  done
done
