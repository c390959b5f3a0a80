set -u
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/r36_pytest.log 2>&1
tail -15 gpurun_out/r36_pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r36_bench128.json 2> gpurun_out/r36_bench128.err
timeout 900 python bench.py --workload c2_2d2048 --no-cpu-baseline > gpurun_out/r36_bench2048.json 2> gpurun_out/r36_bench2048.err
for f in gpurun_out/r36_bench*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['ms_per_step'], d['gmres_iters'], d['roofline']['frac'], d['config']['setup_s'])"; done
