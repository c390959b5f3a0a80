# generic A/B of library builds ab/lib$V.so: bits against the first, kbench, step times
# usage: VARS="A B" bash tools/experiments/ab_libs.sh
set -u
VARS=${VARS:-A B}
FIRST=${VARS%% *}
for V in $VARS; do
  OKG_LIB=ab/lib$V.so timeout 600 python tools/ab_bits.py gpurun_out/bits_$V.npz > /dev/null 2>&1
  [ $V != $FIRST ] && echo "bits $FIRST vs $V: $(timeout 100 python tools/ab_bits.py --cmp gpurun_out/bits_$FIRST.npz gpurun_out/bits_$V.npz 2>&1 | tail -1)"
done
rm -f gpurun_out/bits_*.npz
for V in $VARS; do
  export OKG_LIB=ab/lib$V.so
  echo "== $V kbench 3D 128: $(timeout 300 python tools/kbench.py 3 128 50 2>&1 | grep -v levels | awk '{printf "%s %s; ", $1, $2}')"
  echo "== $V kbench 3D 400: $(OKG_MIN_COARSE=17576 timeout 300 python tools/kbench.py 3 400 20 2>&1 | grep -v levels | awk '{printf "%s %s; ", $1, $2}')"
  echo "== $V kbench 2D 2048: $(timeout 300 python tools/kbench.py 2 2048 50 2>&1 | grep -v levels | awk '{printf "%s %s; ", $1, $2}')"
done
for rep in 1 2; do for V in $VARS; do
  for WL in c4_3d128 c2_2d2048; do
  r=$(OKG_LIB=ab/lib$V.so timeout 300 python bench.py --workload $WL --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
  echo "step $WL $V rep$rep $r"; done
done; done
for V in $VARS; do
  r=$(OKG_LIB=ab/lib$V.so timeout 600 python bench.py --workload c5_3d800 --steps 3 --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])"); echo "step 400 $V $r"
done
