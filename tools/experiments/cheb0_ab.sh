# Chebyshev start vector fused into the first step (k_tiled L_CHEB0, default) against the separate k_cheb_first (OKG_CHEB0=0)
OKG_CHEB0=0 timeout 600 python tools/ab_bits.py gpurun_out/bits_off.npz > /dev/null 2>&1
OKG_CHEB0=1 timeout 600 python tools/ab_bits.py gpurun_out/bits_on.npz > /dev/null 2>&1
echo "bits: $(timeout 100 python tools/ab_bits.py --cmp gpurun_out/bits_off.npz gpurun_out/bits_on.npz 2>&1 | tail -1)"
rm -f gpurun_out/bits_off.npz gpurun_out/bits_on.npz
for rep in 1 2; do for W in 0 1; do
  for WL in c4_3d128 c2_2d2048; do
  r=$(OKG_CHEB0=$W timeout 300 python bench.py --workload $WL --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
  echo "step $WL cheb0=$W rep$rep $r"; done
done; done
for W in 0 1; do
  r=$(OKG_CHEB0=$W timeout 600 python bench.py --workload c5_3d800 --steps 3 --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])"); echo "step 400 cheb0=$W $r"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
