#!/bin/bash
# ncu evidence per config: launch list of one eager step + full captures of its top kernels (1 GPU).
# Reports stay in /tmp/prof on the box; the summaries (profiles/<tag>_c<cfg>_ncu.{md,json}), the
# launch lists and the source-level hot spots come back in gpurun_out/prof.
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${TAG:-r2}
W=/tmp/prof; mkdir -p $W gpurun_out/prof
P="python tools/profile_step.py"
NCU="ncu --clock-control none --profile-from-start off"
for cfg in ${CFGS:-3 2}; do
  timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
    --log-file $W/c${cfg}_launches.csv $P --config $cfg > $W/c${cfg}_list.log 2>&1
  if [ $cfg = 2 ] || [ $cfg = 1 ]; then
    KS="k_rowsel_tc:0 k_op_digit_ntt:8 k_op_eq_mac_nb4:8 k_xp_nttmac:1 k_op_eq_intt:8 k_pack_planes2:0"
  else
    KS="k_rowsel_tk:0 k_y_to_cts:0 k_xp_nttmac:1 k_op_xp_intt:1 k_op_dcp:10 k_op_digit_ntt:8 k_op_eq_mac_nb4:8 k_op_eq_intt:8 k_pack_planes2:0"
  fi
  reps=""
  for ks in $KS; do
    k=${ks%%:*}; sk=${ks##*:}
    timeout 900 $NCU --set full --import-source on -k regex:"$k" -s $sk -c 1 -o $W/c${cfg}_$k $P --config $cfg \
      > $W/c${cfg}_$k.log 2>&1
    if [ -f $W/c${cfg}_$k.ncu-rep ]; then
      reps="$reps $W/c${cfg}_$k.ncu-rep"
      ncu -i $W/c${cfg}_$k.ncu-rep --page source --csv --print-source sass 2>/dev/null > $W/c${cfg}_${k}_src.csv
      python tools/ncu_hotspots.py $W/c${cfg}_${k}_src.csv 40 > gpurun_out/prof/c${cfg}_${k}_hot.txt 2>&1
    fi
  done
  python tools/ncu_summary.py $W/c${cfg}_launches.csv $reps --tag ${TAG}_c${cfg} > $W/c${cfg}_summary.log 2>&1
  cp profiles/${TAG}_c${cfg}_ncu.md profiles/${TAG}_c${cfg}_ncu.json gpurun_out/prof/ 2>/dev/null
  gzip -c $W/c${cfg}_launches.csv > gpurun_out/prof/c${cfg}_launches.csv.gz
  cp $W/*.log gpurun_out/prof/ 2>/dev/null
done
ls -la gpurun_out/prof
