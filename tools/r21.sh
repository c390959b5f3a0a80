set -u
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/r21_pytest.log 2>&1
OKG_MIN_COARSE=17576 timeout 300 python tools/kbench.py 3 400 20 > gpurun_out/r21_400.log 2>&1
timeout 300 python tools/kbench.py 3 128 50 > gpurun_out/r21_128.log 2>&1
timeout 300 python tools/kbench.py 2 2048 50 > gpurun_out/r21_2048.log 2>&1
tail -15 gpurun_out/r21_pytest.log
for f in gpurun_out/r21_*.log; do echo $f; cat $f; done
