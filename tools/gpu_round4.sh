#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for pdl in 1 0; do for tail in 0 -1; do OKG_PDL=$pdl OKG_TAIL=$tail timeout 300 python tools/profile_step.py 3 128 2 | tail -1; done; done
for pdl in 1 0; do for tail in 0 -1; do OKG_PDL=$pdl OKG_TAIL=$tail timeout 300 python tools/profile_step.py 2 2048 2 | tail -1; done; done
