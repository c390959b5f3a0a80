#!/bin/bash
# ncu --set full of the mid-level kernels of one 3D 128^3 step (after a plain run)
set -u
python tools/profile_step.py 3 128 1 > gpurun_out/mid_plain.log 2>&1 || exit 1
SETUP=$(grep -o 'setup_launches=[0-9]*' gpurun_out/mid_plain.log | cut -d= -f2)
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_tiled<3, 0, 1, 2>" -s 20 -c 1 -o gpurun_out/mid_l1resid python tools/profile_step.py 3 128 1 > gpurun_out/ncu_mid1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:k_mg_down" -s 20 -c 2 -o gpurun_out/mid_down python tools/profile_step.py 3 128 1 > gpurun_out/ncu_mid2.log 2>&1
echo done; tail -2 gpurun_out/ncu_mid1.log gpurun_out/ncu_mid2.log
