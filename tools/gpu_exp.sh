#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for v in libgpir.so libgpir_exp_EXP_NO_DCP.so libgpir_exp_EXP_NO_MAC.so libgpir_exp_EXP_NO_FWD.so libgpir_exp_EXP_NO_DCP_EXP_NO_MAC_EXP_NO_FWD.so; do
  echo "== $v"
  GPIR_LIB=$GRAFT_REPO_ROOT/paper_2604_04696_b200/$v timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | grep -o '"phases_ms[^}]*}'
done
