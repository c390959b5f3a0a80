set -u
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_coarse.py -x -q ) > gpurun_out/r29_pytest.log 2>&1
timeout 900 python bench.py --workload c5_3d800 --steps 3 --no-cpu-baseline > gpurun_out/r29_bench400.json 2> gpurun_out/r29_bench400.err
tail -3 gpurun_out/r29_pytest.log
for f in gpurun_out/r29_bench*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['ms_per_step'], d['gmres_iters'], d['roofline']['frac'])"; done
