set -u
mkdir -p gpurun_out
( timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_coarse.py -x -q ) > gpurun_out/r12_pytest.log 2>&1
for S in -1 2; do
  OKG_STREAM=$S timeout 300 python tools/kbench.py 3 128 50 > gpurun_out/r12_kb128_$S.log 2>&1
  OKG_STREAM=$S OKG_MIN_COARSE=17576 timeout 300 python tools/kbench.py 3 400 20 > gpurun_out/r12_kb400_$S.log 2>&1
  OKG_STREAM=$S timeout 300 python tools/kbench.py 2 2048 50 > gpurun_out/r12_kb2048_$S.log 2>&1
done
tail -5 gpurun_out/r12_pytest.log; for f in gpurun_out/r12_kb*; do echo $f; cat $f; done
