for rep in 1 2; do for R in none 1.0 0.6; do
  if [ $R = none ]; then unset OKG_L2PIN; else export OKG_L2PIN=$R; fi
  r=$(timeout 300 python bench.py --no-cpu-baseline --no-kernels 2>/tmp/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
  echo "step 3d128 l2pin=$R rep$rep $r $(grep L2PIN /tmp/err.txt | head -1)"
done; done
unset OKG_L2PIN
r=$(timeout 300 python bench.py --workload c2_2d2048 --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))"); echo "2d none $r"
r=$(OKG_L2PIN=1.0 timeout 300 python bench.py --workload c2_2d2048 --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))"); echo "2d pin1.0 $r"
r=$(OKG_L2PIN=0.5 timeout 300 python bench.py --workload c2_2d2048 --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))"); echo "2d pin0.5 $r"
