set -u
mkdir -p gpurun_out
for cfg in "-" "128" "128:16" "128:32" "128:64"; do
  M=${cfg%%:*}; C=${cfg#*:}; [ "$C" = "$cfg" ] && C=0
  if [ "$M" = "-" ]; then unset OKG_STREAM_MIN_N; else export OKG_STREAM_MIN_N=$M; fi
  export OKG_STREAM_CHUNK=$C
  echo "== stream=$M chunk=$C"
  OKG_LIB=ab/libS.so OKG_MIN_COARSE=17576 timeout 300 python tools/kbench.py 3 400 20 0 1 2 3 4 7 | tail -n +2
  OKG_LIB=ab/libS.so timeout 300 python tools/kbench.py 3 128 50 0 1 2 3 4 7 | tail -n +2
done > gpurun_out/r44.log 2>&1
cat gpurun_out/r44.log
