#!/bin/bash
# ncu --set full of one kernel family, after a plain run of the same command
# usage: KREGEX=... CMD="python tools/kbench.py 3 128 5 0" bash tools/ncu_full.sh OUTNAME
set -u
mkdir -p gpurun_out
$CMD > gpurun_out/ncu_plain_$1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base ${KBASE:-function} -k "regex:${KREGEX}" -s ${SKIP:-3} -c ${COUNT:-1} \
  -o gpurun_out/$1 $CMD > gpurun_out/ncu_$1.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_$1.log
