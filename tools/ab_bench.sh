#!/bin/bash
# A/B of libokg builds (ab/lib$V.so) on the default bench workload: ms per step
# per variant, interleaved reps; then the GPU parity tests against each variant.
# usage: VARS="A B" REPS=3 [TESTS="tests/..."] bash tools/ab_bench.sh OUT [bench args...]
set -u
mkdir -p gpurun_out
OUT=$1; shift
for rep in $(seq ${REPS:-3}); do for V in ${VARS:-A B}; do
  r=$(OKG_LIB=ab/lib$V.so timeout 300 python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,2), d['gmres_iters'])")
  echo "$V rep$rep $r"
done; done > gpurun_out/$OUT.log 2>&1
if [ -n "${TESTS:-}" ]; then for V in ${VARS:-A B}; do
  echo "== tests $V: $(OKG_LIB=ab/lib$V.so timeout 600 python -m pytest $TESTS -m gpu -x -q 2>&1 | tail -n 1)" >> gpurun_out/$OUT.log
done; fi
cat gpurun_out/$OUT.log
