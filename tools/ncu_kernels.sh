#!/bin/bash
# ncu --set full of the fine-level residual sweep (top of the 3D launch lists), the two
# pre-sweeps from zero and the prolongation-staged sweep at 128^3 and 400^3, and of the 2D
# Chebyshev step (top of the 2D launch list) at 2048^2: the 4th launch of the kernel inside
# okg_kernel_timing (after its 3 warm-up launches).
# usage: bash tools/ncu_kernels.sh PREFIX
set -u
P=${1:-m}
run() {  # tag kbench-id dim n load epi [env]
  local RX="k_tiled<.int.$3, .int.$5, .int.$6, .int.8,"
  env ${7:-X=1} KBASE=demangled KREGEX="$RX" SKIP=3 COUNT=1 CMD="python tools/kbench.py $3 $4 5 $2" bash tools/ncu_full.sh ${P}_${1}$4 > /dev/null 2>&1
  local f=${P}_${1}$4
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$f.ncu-rep --page details --csv > gpurun_out/${f}_details.csv 2>/dev/null
  tail -2 gpurun_out/ncu_$f.log
  rm -f gpurun_out/$f.ncu-rep  # ~20 MB each; gpurun brings back at most 64 MiB -- the CSV pages are kept
}
for spec in "resid 1 0 1" "pre2 2 1 2" "prolong 7 2 2"; do
  set -- $spec
  run $1 $2 3 128 $3 $4
  run $1 $2 3 400 $3 $4 OKG_MIN_COARSE=17576
done
run cheb 4 2 2048 0 5
