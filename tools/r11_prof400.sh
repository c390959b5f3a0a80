set -u
mkdir -p gpurun_out
export OKG_MIN_COARSE=17576
OKG_MIN_COARSE=17576 bash tools/launch_list.sh r11_3d400 3 400 > gpurun_out/r11_ll.log 2>&1
KREGEX="k_tiled" SKIP=3 COUNT=1 CMD="python tools/kbench.py 3 400 5 0" bash tools/ncu_full.sh r11_smooth400 > /dev/null 2>&1
ncu -i gpurun_out/r11_smooth400.ncu-rep --page raw --csv > gpurun_out/r11_smooth400_raw.csv 2>/dev/null
ncu -i gpurun_out/r11_smooth400.ncu-rep --page details --csv > gpurun_out/r11_smooth400_details.csv 2>/dev/null
rm -f gpurun_out/r11_smooth400.ncu-rep.bak
head -60 gpurun_out/ll_r11_3d400.summary.txt
