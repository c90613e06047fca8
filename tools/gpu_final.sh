#!/bin/bash
# round-end evidence: GPU suite, smoke, bench lines (config 3 both arms, config 2, 4), ncu evidence per config
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
( nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv; nproc; lscpu | grep "Model name" ) > gpurun_out/z_env.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/z_gputest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/z_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/z_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/z_smoke.txt
timeout 900 python bench.py --impl reference --steps ${RSTEPS:-5} --warmup 1 > gpurun_out/z_ref3.json 2> gpurun_out/z_ref3.err
timeout 900 python bench.py > gpurun_out/z_b3.json 2> gpurun_out/z_b3.err
timeout 600 python bench.py --config 2 > gpurun_out/z_b2.json 2> gpurun_out/z_b2.err
timeout 900 python bench.py --config 4 --no-cpu --steps 5 > gpurun_out/z_b4.json 2> gpurun_out/z_b4.err
CFGS="${PCFGS:-3 2}" TAG=${TAG:-r2f} bash tools/gpu_prof_r2.sh > gpurun_out/z_prof.log 2>&1
