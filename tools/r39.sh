set -u
mkdir -p gpurun_out
for C in 0 -1 5000; do OKG_COLLAPSE=$C timeout 300 python tools/profile_step.py 3 128 3 > gpurun_out/r39_c$C.log 2>&1; done
for C in 0 -1 4500; do OKG_COLLAPSE=$C timeout 300 python tools/profile_step.py 2 2048 3 > gpurun_out/r39_2d_c$C.log 2>&1; done
OKG_COLLAPSE=-1 OKG_MIN_COARSE=17576 timeout 300 python tools/profile_step.py 3 400 2 > gpurun_out/r39_400.log 2>&1
cat gpurun_out/r39_*.log
