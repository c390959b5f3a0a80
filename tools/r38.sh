set -u
mkdir -p gpurun_out
bash tools/launch_list.sh r38_3d128 3 128 > /dev/null 2>&1
grep -i "coarse_sym\|tail\|mg_down\|mg_up" gpurun_out/ll_r38_3d128.summary.txt
head -3 gpurun_out/ll_r38_3d128.summary.txt
