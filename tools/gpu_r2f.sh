#!/bin/bash
# round 2: full GPU suite + the new bench on configs 3 (default, with the reference sample), 2, 4, 5 and the
# sharded orchestration on one GPU
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nproc > gpurun_out/f_env.txt; nvidia-smi --query-gpu=name,memory.total --format=csv >> gpurun_out/f_env.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/f_gputest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/f_gputest.txt
timeout 900 python bench.py > gpurun_out/f_b3.json 2> gpurun_out/f_b3.err; echo "rc=$?" >> gpurun_out/f_b3.err
timeout 600 python bench.py --config 2 --no-cpu > gpurun_out/f_b2.json 2> gpurun_out/f_b2.err; echo "rc=$?" >> gpurun_out/f_b2.err
timeout 900 python bench.py --config 4 --no-cpu --steps 5 > gpurun_out/f_b4.json 2> gpurun_out/f_b4.err; echo "rc=$?" >> gpurun_out/f_b4.err
timeout 1200 python bench.py --config 5 --no-cpu --steps 3 > gpurun_out/f_b5.json 2> gpurun_out/f_b5.err; echo "rc=$?" >> gpurun_out/f_b5.err
timeout 600 python bench.py --config 2 --no-cpu --steps 5 --strategy rowshard > gpurun_out/f_rs2.json 2> gpurun_out/f_rs2.err; echo "rc=$?" >> gpurun_out/f_rs2.err
timeout 600 python bench.py --config 2 --no-cpu --steps 5 --strategy colshard > gpurun_out/f_cs2.json 2> gpurun_out/f_cs2.err; echo "rc=$?" >> gpurun_out/f_cs2.err
