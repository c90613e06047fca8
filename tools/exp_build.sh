#!/bin/bash
# build experiment variants of libgpir (timing only; results are wrong by design)
cd /root/repo
F="-shared -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr"
for v in "$@"; do
  name=$(echo $v | tr ',' '_')
  defs=""; for d in $(echo $v | tr ',' ' '); do defs="$defs -D$d"; done
  nvcc $F $defs -o paper_2604_04696_b200/libgpir_exp_$name.so paper_2604_04696_b200/csrc/gpir.cu &
done
wait
