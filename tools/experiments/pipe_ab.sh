#!/bin/bash
# A/B of the persistent TMA-fed tiled kernels (okg_pipe.cuh) against the one-tile-per-CTA
# kernels: bit identity, per-kernel timings, step times.  usage: bash tools/pipe_ab.sh TAG
set -u
T=${1:-pipe}
mkdir -p gpurun_out
OKG_PIPE=0 timeout 600 python tools/ab_bits.py gpurun_out/${T}_bits_off.npz > gpurun_out/${T}_bits.log 2>&1
OKG_PIPE=1 timeout 600 python tools/ab_bits.py gpurun_out/${T}_bits_on.npz >> gpurun_out/${T}_bits.log 2>&1
timeout 100 python tools/ab_bits.py --cmp gpurun_out/${T}_bits_off.npz gpurun_out/${T}_bits_on.npz >> gpurun_out/${T}_bits.log 2>&1
rm -f gpurun_out/${T}_bits_off.npz gpurun_out/${T}_bits_on.npz
tail -3 gpurun_out/${T}_bits.log
for P in 0 1; do
  echo "== kbench 3D 128 pipe=$P"; OKG_PIPE=$P timeout 300 python tools/kbench.py 3 128 50 2>&1 | tail -9
  echo "== kbench 3D 400 pipe=$P"; OKG_MIN_COARSE=17576 OKG_PIPE=$P timeout 300 python tools/kbench.py 3 400 20 2>&1 | tail -9
  echo "== kbench 2D 2048 pipe=$P"; OKG_PIPE=$P timeout 300 python tools/kbench.py 2 2048 50 2>&1 | tail -9
done
for rep in 1 2; do for P in 0 1; do
  for W in c4_3d128 c2_2d2048; do
    r=$(OKG_PIPE=$P timeout 300 python bench.py --workload $W --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])")
    echo "step $W pipe=$P rep$rep $r"
  done
done; done
r=$(OKG_PIPE=0 timeout 600 python bench.py --workload c5_3d800 --steps 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])"); echo "step 400 pipe=0 $r"
r=$(OKG_PIPE=1 timeout 600 python bench.py --workload c5_3d800 --steps 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])"); echo "step 400 pipe=1 $r"
