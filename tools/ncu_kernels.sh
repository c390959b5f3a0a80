#!/bin/bash
# ncu --set full of the fine-level residual sweep (top of the launch lists), the two
# pre-sweeps from zero and the prolongation-staged sweep, at 128^3 and 400^3: the 4th
# launch of the kernel inside okg_kernel_timing (after its 3 warm-up launches).
# usage: bash tools/ncu_kernels.sh PREFIX
set -u
P=${1:-m}
for spec in "resid 1 0 1" "pre2 2 1 2" "prolong 7 2 2"; do
  set -- $spec
  RX="k_tiled<.int.3, .int.$3, .int.$4, .int.8,"
  KBASE=demangled KREGEX="$RX" SKIP=3 COUNT=1 CMD="python tools/kbench.py 3 128 5 $2" bash tools/ncu_full.sh ${P}_${1}128 > /dev/null 2>&1
  OKG_MIN_COARSE=17576 KBASE=demangled KREGEX="$RX" SKIP=3 COUNT=1 CMD="python tools/kbench.py 3 400 5 $2" bash tools/ncu_full.sh ${P}_${1}400 > /dev/null 2>&1
  for f in ${P}_${1}128 ${P}_${1}400; do
    ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
    ncu -i gpurun_out/$f.ncu-rep --page details --csv > gpurun_out/${f}_details.csv 2>/dev/null
    tail -2 gpurun_out/ncu_$f.log
    rm -f gpurun_out/$f.ncu-rep  # ~20 MB each; gpurun brings back at most 64 MiB -- the CSV pages are kept
  done
done
