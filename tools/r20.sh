set -u
mkdir -p gpurun_out
export OKG_MIN_COARSE=17576
timeout 300 python tools/kbench.py 3 400 20 > gpurun_out/r20_400.log 2>&1
OKG_DBG_NOBND=1 timeout 300 python tools/kbench.py 3 400 20 > gpurun_out/r20_400nb.log 2>&1
timeout 300 python tools/kbench.py 3 128 50 > gpurun_out/r20_128.log 2>&1
OKG_DBG_NOBND=1 timeout 300 python tools/kbench.py 3 128 50 > gpurun_out/r20_128nb.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r20_bench128.json 2>&1
timeout 900 python bench.py --workload c5_3d800 --steps 3 --no-cpu-baseline > gpurun_out/r20_bench400.json 2>&1
for f in gpurun_out/r20_*.log; do echo $f; cat $f; done
for f in gpurun_out/r20_bench*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d['ms_per_step'], d['gmres_iters'])"; done
