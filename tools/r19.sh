set -u
mkdir -p gpurun_out
export OKG_MIN_COARSE=17576
for TI in 8 4; do for C in 30 40 50 60; do echo "TI=$TI carve=$C"; OKG_DBG_TI=$TI OKG_DBG_CARVE=$C OKG_DBG_CARVEC=$C timeout 300 python tools/kbench.py 3 400 20 | tail -8; done; done > gpurun_out/r19_400.log 2>&1
for TI in 8 4; do for C in 30 50 100; do echo "TI=$TI carve=$C"; OKG_DBG_TI=$TI OKG_DBG_CARVE=$C OKG_DBG_CARVEC=$C timeout 300 python tools/kbench.py 3 128 50 | tail -8; done; done > gpurun_out/r19_128.log 2>&1
for TI in 8 4; do for C in 30 50 100; do echo "TI=$TI carve=$C"; OKG_DBG_TI=$TI OKG_DBG_CARVE=$C OKG_DBG_CARVEC=$C timeout 300 python tools/kbench.py 2 2048 50 | tail -8; done; done > gpurun_out/r19_2048.log 2>&1
cat gpurun_out/r19_*.log
