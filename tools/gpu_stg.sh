#!/bin/bash
# staged-digit external-product kernel A/B (GPIR_XP_STAGED): parity + config 3/2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
GPIR_XP_STAGED=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "expand_stages or subs or pipeline or config2 or interleaved or golden" > gpurun_out/stg_test.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/stg_test.txt
for e in 1 0; do for cfg in 3 2; do
  GPIR_XP_STAGED=$e timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --material uniform > gpurun_out/stg_${cfg}_$e.json 2> gpurun_out/stg_${cfg}_$e.err
done; done
