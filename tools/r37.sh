set -u
mkdir -p gpurun_out
for C in 0 -1; do OKG_COLLAPSE=$C timeout 300 python tools/profile_step.py 3 128 3 > gpurun_out/r37_c$C.log 2>&1; done
for C in 0 -1; do OKG_COLLAPSE=$C timeout 300 python tools/profile_step.py 2 2048 3 > gpurun_out/r37_2d_c$C.log 2>&1; done
cat gpurun_out/r37_*.log
