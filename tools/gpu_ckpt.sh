#!/bin/bash
# checkpoint: bench lines (config 2 default, config 3), reference arm, launch list, full captures
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-ck}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-300
timeout 900 python bench.py --config 3 --no-cpu --steps 5 > gpurun_out/bench3_${TAG}.log 2>&1; echo "bench3 rc=$?"; tail -1 gpurun_out/bench3_${TAG}.log | cut -c1-600
timeout 300 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref_${TAG}.log 2>&1; echo "ref rc=$?"
B="python bench.py --steps 1 --warmup 3 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $B > /dev/null 2>&1; echo "list rc=$?"
for k in ${FULLKS:-k_rowsel_tc k_eq_nttmac}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/full_${TAG}_$k $B > /dev/null 2>&1
  echo "$k rc=$?"
done
du -sh gpurun_out
