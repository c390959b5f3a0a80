set -u
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k "regex:k_vcycle_tail|k_mg_down" -s 30 -c 3 -o gpurun_out/r35_mid python tools/profile_step.py 3 128 1 > gpurun_out/r35_mid.log 2>&1
for F in 0 1 2; do OKG_FUSE=$F timeout 300 python tools/profile_step.py 3 128 3 > gpurun_out/r35_fuse$F.log 2>&1; done
OKG_TAIL=-1 timeout 300 python tools/profile_step.py 3 128 3 > gpurun_out/r35_notail.log 2>&1
tail -2 gpurun_out/r35_fuse*.log gpurun_out/r35_notail.log
