# quick A/B of library builds ab/lib$V.so: bits against the first, then step times (3 reps)
VARS=${VARS:-A B}
FIRST=${VARS%% *}
for V in $VARS; do
  OKG_LIB=ab/lib$V.so timeout 600 python tools/ab_bits.py gpurun_out/bits_$V.npz > /dev/null 2>&1
  [ $V != $FIRST ] && echo "bits $FIRST vs $V: $(timeout 100 python tools/ab_bits.py --cmp gpurun_out/bits_$FIRST.npz gpurun_out/bits_$V.npz 2>&1 | tail -1)"
done
rm -f gpurun_out/bits_*.npz
for rep in 1 2 3; do for V in $VARS; do for WL in c4_3d128 c2_2d2048; do
  r=$(OKG_LIB=ab/lib$V.so timeout 300 python bench.py --workload $WL --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
  echo "step $WL $V rep$rep $r"; done; done; done
bash tools/experiments/level_kbench.sh
