#!/bin/bash
# the sharded bench paths on one GPU (identity collectives): config 3 row shards, config 4 column shards (compact, windows)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --config 3 --strategy rowshard --no-cpu --steps 3 > gpurun_out/s_rs3.json 2> gpurun_out/s_rs3.err; echo "rc=$?" >> gpurun_out/s_rs3.err
timeout 1200 python bench.py --config 4 --strategy colshard --no-cpu --steps 2 > gpurun_out/s_cs4.json 2> gpurun_out/s_cs4.err; echo "rc=$?" >> gpurun_out/s_cs4.err
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "cluster or capacity" > gpurun_out/s_test.txt 2>&1; echo "rc=$?" >> gpurun_out/s_test.txt
