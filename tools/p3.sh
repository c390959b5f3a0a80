set -u
mkdir -p gpurun_out
OKG_PIPE=1 timeout 120 python tools/kbench.py 3 64 20 > gpurun_out/p3_kb64_pipe.log 2>&1; echo "kb64 rc=$?"; cat gpurun_out/p3_kb64_pipe.log
OKG_PIPE=0 timeout 300 python tools/ab_bits.py gpurun_out/p3_A.npz > gpurun_out/p3_A.log 2>&1; echo "A rc=$?"
OKG_PIPE=1 timeout 300 python tools/ab_bits.py gpurun_out/p3_B.npz > gpurun_out/p3_B.log 2>&1; echo "B rc=$?"; tail -3 gpurun_out/p3_B.log
python tools/ab_bits.py --cmp gpurun_out/p3_A.npz gpurun_out/p3_B.npz
for P in 0 1; do echo "== PIPE=$P"; OKG_PIPE=$P timeout 300 python tools/kbench.py 3 128 50; done
for P in 0 1; do echo "== PIPE=$P 2d"; OKG_PIPE=$P timeout 300 python tools/kbench.py 2 2048 50; done
for P in 0 1 0 1; do echo "== bench PIPE=$P: $(OKG_PIPE=$P timeout 300 python bench.py --no-cpu-baseline --no-kernels --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'])")"; done
OKG_PIPE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
