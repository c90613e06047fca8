#!/bin/bash
# round 2: RowSel (k_rowsel_tk + k_y_to_cts) parity subset, config 3 timing, ncu full captures of both
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rowsel or config or interleaved or pipeline or graph" > gpurun_out/e_gputest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/e_gputest.txt
B="python bench.py --steps 5 --warmup 3 --no-cpu --material uniform"
timeout 600 $B --config 3 > gpurun_out/e_b3.json 2> gpurun_out/e_b3.err
P="python bench.py --steps 1 --warmup 3 --no-cpu --material uniform --config 3"
for k in k_rowsel_tk k_y_to_cts; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/r2e_$k $P > gpurun_out/e_ncu_$k.log 2>&1
done
