#!/bin/bash
# RowSel kernel iteration: parity subset + config 3 / 4 timing + tk profile counters
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rowsel or config or capacity or interleaved or graph or dropin" > gpurun_out/tk_test.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/tk_test.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --material uniform > gpurun_out/tkb.json 2> gpurun_out/tkb.err
GPIR_TC_PROF=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --material uniform > gpurun_out/tkp.json 2> gpurun_out/tkp.err
