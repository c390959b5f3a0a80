#!/bin/bash
# warm launch list of one Newton step: plain run first, then ncu (gpu__time_duration per
# kernel, no cache flush, no clock control) skipping the setup kernels.
# usage: bash tools/launch_list.sh OUTNAME DIM N   (env OKG_* knobs pass through)
set -u
mkdir -p gpurun_out
python tools/profile_step.py $2 $3 1 > gpurun_out/ll_plain_$1.log 2>&1 || { cat gpurun_out/ll_plain_$1.log; exit 1; }
cat gpurun_out/ll_plain_$1.log
SETUP=$(grep -o 'setup_launches=[0-9]*' gpurun_out/ll_plain_$1.log | cut -d= -f2)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv \
  --log-file gpurun_out/ll_$1.csv python tools/profile_step.py $2 $3 1 > gpurun_out/ll_ncu_$1.log 2>&1
echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/ll_$1.csv 45 > gpurun_out/ll_$1.summary.txt
head -50 gpurun_out/ll_$1.summary.txt
