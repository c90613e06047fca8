#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rowsel or pipeline" > gpurun_out/pytest_rowsel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rowsel.log
tail -2 gpurun_out/pytest_rowsel.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/bench.log | cut -c1-900
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_rowsel_tc|k_pack" -s 0 -c 6 python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_tc.txt 2>&1
grep -E "k_rowsel_tc|k_pack|duration|dram__bytes|tensor|pipe_tc" gpurun_out/ncu_tc.txt | head -40
