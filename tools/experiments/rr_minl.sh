for rep in 1 2; do for ML in 9 1 2; do
  r=$(OKG_RR_MINL=$ML timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
  echo "step 3d128 rr_minl=$ML rep$rep $r"
done; done
