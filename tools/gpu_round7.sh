#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python tools/profile_step.py 3 128 2 | tail -1; python tools/profile_step.py 2 2048 2 | tail -1
python tools/profile_step.py 3 128 1 > gpurun_out/pp.log 2>&1 && S=$(grep setup_launches gpurun_out/pp.log | cut -d= -f2) && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s $S --csv \
  --log-file gpurun_out/launches_warm.csv python tools/profile_step.py 3 128 1 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
KREGEX="k_tiled" CMD="python tools/kbench.py 3 128 5 0" SKIP=3 COUNT=1 bash tools/ncu_full.sh smooth3d_r7
