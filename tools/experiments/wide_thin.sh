OKG_WIDE=0 timeout 600 python tools/ab_bits.py gpurun_out/bits_off.npz > /dev/null 2>&1
OKG_WIDE=3 timeout 600 python tools/ab_bits.py gpurun_out/bits_on.npz > /dev/null 2>&1
echo "bits: $(timeout 100 python tools/ab_bits.py --cmp gpurun_out/bits_off.npz gpurun_out/bits_on.npz 2>&1 | tail -1)"
rm -f gpurun_out/bits_off.npz gpurun_out/bits_on.npz
for rep in 1 2; do for W in 2 3; do
  for WL in c4_3d128 c2_2d2048; do
  r=$(OKG_WIDE=$W timeout 300 python bench.py --workload $WL --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
  echo "step $WL wide=$W rep$rep $r"; done
done; done
for W in 2 3; do
  r=$(OKG_WIDE=$W timeout 600 python bench.py --workload c5_3d800 --steps 3 --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])"); echo "step 400 wide=$W $r"
done
