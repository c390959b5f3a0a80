set -u
mkdir -p gpurun_out
(nproc; free -g; grep -m1 "model name" /proc/cpuinfo; nvidia-smi -L; python -c "import torch;print(torch.__version__)") > gpurun_out/p1_host.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/p1_bench.json 2> gpurun_out/p1_bench.err
timeout 600 python tools/instep_kernels.py 3 128 1 45 > gpurun_out/p1_instep.txt 2>&1
cat gpurun_out/p1_host.txt; tail -c 1500 gpurun_out/p1_bench.json; head -30 gpurun_out/p1_instep.txt
