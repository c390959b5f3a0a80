set -u
mkdir -p gpurun_out
OKG_PIPE16=0 timeout 300 python tools/ab_bits.py /tmp/p9_A.npz > gpurun_out/p9_A.log 2>&1; echo "A rc=$?"
OKG_PIPE16=1 timeout 300 python tools/ab_bits.py /tmp/p9_B.npz > gpurun_out/p9_B.log 2>&1; echo "B rc=$?"; tail -2 gpurun_out/p9_B.log
python tools/ab_bits.py --cmp /tmp/p9_A.npz /tmp/p9_B.npz
for P in 0 1; do echo "== PIPE16=$P"; OKG_PIPE16=$P timeout 300 python tools/kbench.py 3 128 50 | tail -n +2; done
for P in 0 1; do echo "== PIPE16=$P 2d"; OKG_PIPE16=$P timeout 300 python tools/kbench.py 2 2048 50 | tail -n +2; done
for P in 0 1 0 1; do echo "== bench PIPE16=$P: $(OKG_PIPE16=$P timeout 300 python bench.py --no-cpu-baseline --no-kernels --steps 10 2>gpurun_out/p9_bench_err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'])")"; done
for P in 0 1; do echo "== bench 2D PIPE16=$P: $(OKG_PIPE16=$P timeout 300 python bench.py --workload c2_2d2048 --no-cpu-baseline --no-kernels --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'])")"; done
OKG_PIPE16=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
OKG_PIPE16=1 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_tiled_p" -s 3 -c 1 -o gpurun_out/p9_resid3d python tools/kbench.py 3 128 20 1 > gpurun_out/p9_ncu3.log 2>&1; echo "ncu rc=$?"
