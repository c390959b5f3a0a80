set -u
mkdir -p gpurun_out
OKG_MIN_COARSE=17576 timeout 300 python tools/kbench.py 3 400 20 > gpurun_out/r22_400.log 2>&1
timeout 300 python tools/kbench.py 3 128 50 > gpurun_out/r22_128.log 2>&1
timeout 300 python tools/kbench.py 2 2048 50 > gpurun_out/r22_2048.log 2>&1
( timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/r22_pytest.log 2>&1
tail -3 gpurun_out/r22_pytest.log
for f in gpurun_out/r22_*.log; do echo $f; cat $f; done
