#!/bin/bash
# gpu_quick + launch list (+ full capture of $FULLK) in one call
cd "$GRAFT_REPO_ROOT" || exit 1
bash tools/gpu_quick.sh
bash tools/gpu_list.sh
