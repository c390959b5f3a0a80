for FN in 0 32 64; do
  for rep in 1 2; do
  r=$(OKG_FUSE_DOWN_N=$FN timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
  echo "step 3D128 fuse_down_n=$FN rep$rep $r"; done
done
for FN in 0 1024; do
  r=$(OKG_FUSE_DOWN_N=$FN timeout 300 python bench.py --workload c2_2d2048 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
  echo "step 2D2048 fuse_down_n=$FN $r"
done
OKG_FUSE_DOWN_N=0 timeout 600 python tools/ab_bits.py gpurun_out/bits_off.npz > /dev/null 2>&1
OKG_FUSE_DOWN_N=64 timeout 600 python tools/ab_bits.py gpurun_out/bits_on.npz > /dev/null 2>&1
echo "bits: $(timeout 100 python tools/ab_bits.py --cmp gpurun_out/bits_off.npz gpurun_out/bits_on.npz 2>&1 | tail -1)"
rm -f gpurun_out/bits_off.npz gpurun_out/bits_on.npz
