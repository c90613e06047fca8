#!/bin/bash
# ncu launch list of one bench step (+ optional full capture of kernel regex $FULLK)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-x}
B="python bench.py --steps 1 --warmup 3 --no-cpu ${BENCH_ARGS}"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_list_$TAG.log 2>&1
echo "list rc=$?"
if [ -n "$FULLK" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$FULLK -s ${SKIPK:-2} -c 1 -o gpurun_out/full_${TAG} $B > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "full rc=$?"
fi
