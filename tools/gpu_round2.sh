#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for spec in "3 128" "2 2048"; do timeout 120 python tools/kbench.py $spec 50; done
timeout 300 python tools/profile_step.py 3 128 3
timeout 300 python tools/profile_step.py 2 2048 3
if [ "${NCUFULL:-1}" = "1" ]; then
KREGEX="k_tiled" CMD="python tools/kbench.py 3 128 5 0" SKIP=3 COUNT=1 bash tools/ncu_full.sh smooth3d
fi
