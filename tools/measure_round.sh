#!/bin/bash
# round measurement refresh: bench lines (3D 128^3, 400^3 slice of 800^3, 2D 2048^2,
# reference arm), per-step launch lists, ncu --set full of the dominant kernel
set -u
mkdir -p gpurun_out
P=${PFX:-m}
timeout 900 python bench.py > gpurun_out/${P}_bench_3d128.json 2> gpurun_out/${P}_bench_3d128.err
timeout 900 python bench.py --workload c5_3d800 --steps 3 > gpurun_out/${P}_bench_3d400.json 2> gpurun_out/${P}_bench_3d400.err
timeout 900 python bench.py --workload c2_2d2048 --no-cpu-baseline > gpurun_out/${P}_bench_2d2048.json 2> gpurun_out/${P}_bench_2d2048.err
timeout 900 python bench.py --impl reference > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err
bash tools/launch_list.sh ${P}_3d128 3 128 > /dev/null 2>&1
OKG_MIN_COARSE=17576 bash tools/launch_list.sh ${P}_3d400 3 400 > /dev/null 2>&1
bash tools/launch_list.sh ${P}_2d2048 2 2048 > /dev/null 2>&1
bash tools/ncu_kernels.sh ${P}
for f in gpurun_out/${P}_bench_*.json; do echo $f; tail -c 400 $f; echo; done
head -12 gpurun_out/ll_${P}_3d128.summary.txt gpurun_out/ll_${P}_3d400.summary.txt gpurun_out/ll_${P}_2d2048.summary.txt
