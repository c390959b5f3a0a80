# A/B of two libokg builds on one box: bash tools/ab.sh OUT "kbench args"...
set -u
mkdir -p gpurun_out
OUT=$1; shift
for rep in 1 2; do for V in ${VARS:-A B}; do for args in "$@"; do
  echo "== $V $args"; OKG_LIB=ab/lib$V.so OKG_MIN_COARSE=17576 timeout 300 python tools/kbench.py $args | tail -n +2
done; done; done > gpurun_out/$OUT.log 2>&1
cat gpurun_out/$OUT.log
