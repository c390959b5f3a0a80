set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edge.py tests/test_cpp_api.py -x -q > gpurun_out/p2_edge.log 2>&1
tail -15 gpurun_out/p2_edge.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/p2_bench.json 2> gpurun_out/p2_bench.err
tail -c 3000 gpurun_out/p2_bench.json; tail -5 gpurun_out/p2_bench.err
