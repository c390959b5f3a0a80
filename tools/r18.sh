set -u
mkdir -p gpurun_out
export OKG_MIN_COARSE=17576
for C in 100 75 50 25; do OKG_DBG_CARVE=$C OKG_DBG_NOBND=1 timeout 300 python tools/kbench.py 3 400 20 0 1 2 3 > gpurun_out/r18_c$C.log 2>&1; done
for f in gpurun_out/r18_*; do echo $f; cat $f; done
