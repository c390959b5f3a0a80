set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r9_smi.txt 2>&1
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/r9_pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r9_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r9_bench_3d128.json 2> gpurun_out/r9_bench_3d128.err
tail -3 gpurun_out/r9_pytest_gpu.log; cat gpurun_out/r9_smoke.log | tail -2; tail -c 400 gpurun_out/r9_bench_3d128.json
