#!/bin/bash
# launch list + full captures of the top kernels for profiles/ (1 GPU)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $B > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
for k in k_rowsel_tc k_eq_fused k_pack_planes; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIPK:-2} -c 1 -o gpurun_out/r1_full_$k $B > gpurun_out/ncu_full_$k.log 2>&1
  echo "$k rc=$?"
done
