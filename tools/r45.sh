set -u
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -m gpu -x -q -k "residual or newton or golden or oracle or diag" ) > gpurun_out/r45_pytest.log 2>&1
tail -3 gpurun_out/r45_pytest.log
bash tools/launch_list.sh r45_3d128 3 128 > /dev/null 2>&1
OKG_MIN_COARSE=17576 bash tools/launch_list.sh r45_3d400 3 400 > /dev/null 2>&1
grep "k_residual\|total" gpurun_out/ll_r45_3d128.summary.txt gpurun_out/ll_r45_3d400.summary.txt
