#!/bin/bash
# round-1 measurement refresh: bench lines, launch list, ncu of the dominant kernel
set -u
mkdir -p gpurun_out
cd paper_1603_04570_b200/csrc && make -s && cd ../..
timeout 900 python bench.py > gpurun_out/r8_bench_3d128.json 2> gpurun_out/r8_bench_3d128.err
timeout 900 python bench.py --workload c2_2d2048 --no-cpu-baseline > gpurun_out/r8_bench_2d2048.json 2> gpurun_out/r8_bench_2d2048.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r8_bench_ref.json 2> gpurun_out/r8_bench_ref.err
bash tools/launch_list.sh r8_3d128 3 128 > /dev/null 2>&1
KREGEX="k_tiled" SKIP=3 COUNT=1 CMD="python tools/kbench.py 3 128 5 0" bash tools/ncu_full.sh r8_smooth128 > /dev/null 2>&1
ncu -i gpurun_out/r8_smooth128.ncu-rep --page raw --csv > gpurun_out/r8_smooth128_raw.csv 2>/dev/null
tail -c 600 gpurun_out/r8_bench_3d128.json; echo; tail -c 300 gpurun_out/r8_bench_2d2048.json; echo; tail -c 300 gpurun_out/r8_bench_ref.json; echo
head -5 gpurun_out/ll_r8_3d128.summary.txt
