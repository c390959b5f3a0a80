#!/bin/bash
# variants of the pipe kernels (ab/lib$V.so) against the same library with OKG_PIPE=0
set -u
mkdir -p gpurun_out
for V in ${VARS:-A B C}; do
  export OKG_LIB=ab/lib$V.so
  if [ "${BITS:-1}" = "1" ]; then
    OKG_PIPE=0 timeout 600 python tools/ab_bits.py gpurun_out/bits_off.npz > /dev/null 2>&1
    OKG_PIPE=1 timeout 600 python tools/ab_bits.py gpurun_out/bits_on.npz > /dev/null 2>&1
    echo "== $V bits: $(timeout 100 python tools/ab_bits.py --cmp gpurun_out/bits_off.npz gpurun_out/bits_on.npz 2>&1 | tail -1)"
    rm -f gpurun_out/bits_off.npz gpurun_out/bits_on.npz
  fi
  for P in ${PIPES:-1}; do
    echo "== $V kbench 3D 128 pipe=$P"; OKG_PIPE=$P timeout 300 python tools/kbench.py 3 128 50 2>&1 | grep -v levels
    echo "== $V kbench 3D 400 pipe=$P"; OKG_MIN_COARSE=17576 OKG_PIPE=$P timeout 300 python tools/kbench.py 3 400 20 2>&1 | grep -v levels
  done
  for rep in 1 2; do for P in 0 1; do
    r=$(OKG_PIPE=$P timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
    echo "step $V 128 pipe=$P rep$rep $r"
  done; done
done
