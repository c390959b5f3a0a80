set -u
mkdir -p gpurun_out
export OKG_MIN_COARSE=17576
timeout 600 ncu --set full --clock-control none -k "regex:k_tiled" -s 3 -c 1 -o gpurun_out/r15_prod python tools/kbench.py 3 400 5 0 > gpurun_out/r15_prod.log 2>&1
timeout 600 ncu --set full --clock-control none -k "regex:v4_tile_async" -s 6 -c 1 -o gpurun_out/r15_mb ./tools/stencil_bench 400 > gpurun_out/r15_mb.log 2>&1
for f in r15_prod r15_mb; do ncu -i gpurun_out/$f.ncu-rep --page details --csv > gpurun_out/${f}_details.csv 2>/dev/null; ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null; done
ls -la gpurun_out/r15*
