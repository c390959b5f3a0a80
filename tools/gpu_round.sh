#!/bin/bash
# one gpurun call: GPU tests, bench, plain run + ncu launch list of one Newton step
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json | head -c 3000; echo
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 python tools/profile_step.py ${PDIM:-3} ${PN:-128} 1 > gpurun_out/profile_plain.log 2>&1; rc=$?
  echo "plain rc=$rc"; cat gpurun_out/profile_plain.log
  S=$(grep setup_launches gpurun_out/profile_plain.log | cut -d= -f2)
  if [ $rc -eq 0 ]; then
    timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s $S --csv \
      --log-file gpurun_out/launches.csv python tools/profile_step.py ${PDIM:-3} ${PN:-128} 1 > gpurun_out/ncu.log 2>&1
    echo "ncu rc=$?"; tail -2 gpurun_out/ncu.log
  fi
fi
if [ "${PROBE:-0}" = "1" ]; then timeout 600 python tools/gpu_probe.py --big ${BIG:-3:64,2:512,3:128,2:2048} > gpurun_out/probe.log 2>&1; echo "probe rc=$?"; grep -E "timing|step" gpurun_out/probe.log | tail -20; fi
