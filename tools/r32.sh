set -u
mkdir -p gpurun_out
export OKG_MIN_COARSE=17576
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_tiled" -s 3 -c 1 -o gpurun_out/r32_pre2 python tools/kbench.py 3 400 5 2 > gpurun_out/r32_pre2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_tiled" -s 3 -c 1 -o gpurun_out/r32_smooth python tools/kbench.py 3 400 5 0 > gpurun_out/r32_smooth.log 2>&1
ls -la gpurun_out/r32*
