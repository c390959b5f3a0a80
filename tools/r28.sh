set -u
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/r28_pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/r28_bench128.json 2> gpurun_out/r28_bench128.err
timeout 900 python bench.py --workload c5_3d800 --steps 3 --no-cpu-baseline > gpurun_out/r28_bench400.json 2> gpurun_out/r28_bench400.err
OKG_MIN_COARSE=17576 bash tools/launch_list.sh r28_3d400 3 400 > /dev/null 2>&1
bash tools/launch_list.sh r28_3d128 3 128 > /dev/null 2>&1
tail -3 gpurun_out/r28_pytest.log
for f in gpurun_out/r28_bench*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['ms_per_step'], d['gmres_iters'], d['roofline']['frac'])"; done
head -30 gpurun_out/ll_r28_3d400.summary.txt; head -40 gpurun_out/ll_r28_3d128.summary.txt
