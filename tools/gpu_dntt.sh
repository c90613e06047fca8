#!/bin/bash
# digit NTT with all limbs per CTA: parity + configs 3/2 both ways
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "expand_stages or subs or pipeline or config or interleaved or golden" > gpurun_out/dn_test.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/dn_test.txt
for e in 1 0; do for cfg in 3 2; do
  GPIR_DNTT_ALL=$e timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --material uniform > gpurun_out/dn_${cfg}_$e.json 2> gpurun_out/dn_${cfg}_$e.err
done; done
