set -u
mkdir -p gpurun_out
export OKG_MIN_COARSE=17576
timeout 300 python tools/kbench.py 3 400 20 0 1 2 3 > gpurun_out/r17_a.log 2>&1
OKG_DBG_NOBND=1 timeout 300 python tools/kbench.py 3 400 20 0 1 2 3 > gpurun_out/r17_b.log 2>&1
OKG_DBG_NOBND=1 timeout 300 python tools/kbench.py 3 128 50 0 1 2 3 > gpurun_out/r17_c.log 2>&1
for f in gpurun_out/r17_*; do echo $f; cat $f; done
