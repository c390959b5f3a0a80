# fused residual+restriction (okg_rr.cuh, OKG_RR=1) against the two separate kernels (OKG_RR=0)
OKG_RR=0 timeout 600 python tools/ab_bits.py gpurun_out/bits_off.npz > /dev/null 2>&1
OKG_RR=1 timeout 600 python tools/ab_bits.py gpurun_out/bits_on.npz > /dev/null 2>&1
echo "bits: $(timeout 100 python tools/ab_bits.py --cmp gpurun_out/bits_off.npz gpurun_out/bits_on.npz 2>&1 | tail -1)"
rm -f gpurun_out/bits_off.npz gpurun_out/bits_on.npz
for rep in 1 2; do for RR in 0 1; do
  for W in c4_3d128 c2_2d2048; do
  r=$(OKG_RR=$RR timeout 300 python bench.py --workload $W --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
  echo "step $W rr=$RR rep$rep $r"; done
done; done
for RR in 0 1; do
  r=$(OKG_RR=$RR timeout 600 python bench.py --workload c5_3d800 --steps 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])"); echo "step 400 rr=$RR $r"
done
