#!/bin/bash
# what the round-end driver runs: GPU tests, smoke, the reference arm and our arm at N=1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/ds_test.txt 2>&1; echo "rc=$?" >> gpurun_out/ds_test.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ds_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/ds_smoke.txt
( time timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/ds_ref.json 2> gpurun_out/ds_ref.err
( time timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/ds_ours.json 2> gpurun_out/ds_ours.err
