set -u
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_parity.py -k "coarse or d2n90big" -x -q ) > gpurun_out/r10_pytest.log 2>&1
timeout 1200 python bench.py --workload c5_3d800 --steps 3 --warmup 3 > gpurun_out/r10_bench_c5.json 2> gpurun_out/r10_bench_c5.err
tail -15 gpurun_out/r10_pytest.log; tail -c 1500 gpurun_out/r10_bench_c5.json; tail -20 gpurun_out/r10_bench_c5.err
