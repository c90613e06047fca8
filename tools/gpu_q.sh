#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for k in ${KERNELS}; do
timeout 300 ncu --section SpeedOfLight --section WarpStateStats --section ComputeWorkloadAnalysis --section Occupancy --section MemoryWorkloadAnalysis --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio --clock-control none -k regex:$k -s ${SKIP:-3} -c 1 python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_q_$k.txt 2>&1
grep -E "Duration|inst_executed|Ipc A|Achieved Occupancy|Registers Per|stalled|L1/TEX Hit|L2 Hit|DRAM Through|Block Limit" gpurun_out/ncu_q_$k.txt | sed "s/^/$k: /"
done
