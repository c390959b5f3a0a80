set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_baseline_full.py tests/test_gpu_edge.py -q -s > gpurun_out/p10_full.log 2>&1; echo "rc=$?"
grep -E "passed|failed|c[234]_" gpurun_out/p10_full.log | cut -c1-400
