#!/bin/bash
# node-batched ExpandQuery MAC: parity of the op-level paths + eq8 per-kernel times for NB in $NBS
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "op or pipeline or execution" 2>&1 | tail -1
for nb in ${NBS:-1 8 16 32}; do echo "NB=$nb"; GPIR_MAC_NB=$nb CHUNKS="0" bash tools/gpu_chunk.sh; done
