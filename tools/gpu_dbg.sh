#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for f in capacity client_gpu cluster dropin_latpir; do
  timeout 900 python -m pytest tests/test_$f.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "not config and (capacity or client or cluster or dropin or rowsel_engines)" > gpurun_out/dbg_$f.txt 2>&1
done
