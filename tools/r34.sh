set -u
mkdir -p gpurun_out
( timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/r34_pytest.log 2>&1
tail -3 gpurun_out/r34_pytest.log
