for TI in 8 7 6 5; do
  echo "== TI=$TI"; OKG_TI=$TI timeout 300 python tools/kbench.py 3 128 50 2>&1 | grep -v levels | tr '\n' ';'; echo
  for rep in 1 2; do
  r=$(OKG_TI=$TI timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
  echo "step 128 TI=$TI rep$rep $r"; done
done
