#!/bin/bash
# RowSel variants at config 3 (B = 128, d1 = 512) and config 2
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 600 python -m pytest tests -x -q -m gpu -k "rowsel or pipeline" 2>&1 | tail -1
for v in "32 0" "32 1" "64 0" "64 1"; do
  set -- $v
  echo "NT=$1 ORDER=$2"
  GPIR_TC_NT=$1 GPIR_TC_ORDER=$2 timeout 300 python bench.py --config 3 --no-cpu --steps 3 --warmup 3 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']),d['phases_ms']['RowSel'],d['roofline']['frac'])"
done
python bench.py --no-cpu --steps 20 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cfg2',round(d['value']),d['phases_ms']['RowSel'],d['roofline']['frac'])"
