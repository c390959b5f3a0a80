set -u
mkdir -p gpurun_out
OKG_PIPE=0 timeout 300 python tools/ab_bits.py /tmp/p4_A.npz > gpurun_out/p4_A.log 2>&1; echo "A rc=$?"
OKG_PIPE=1 timeout 300 python tools/ab_bits.py /tmp/p4_B.npz > gpurun_out/p4_B.log 2>&1; echo "B rc=$?"; tail -3 gpurun_out/p4_B.log
python tools/ab_bits.py --cmp /tmp/p4_A.npz /tmp/p4_B.npz
OKG_PIPE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/p4_parity.log 2>&1; tail -30 gpurun_out/p4_parity.log
OKG_PIPE=1 timeout 300 python tools/kbench.py 2 2048 20 1 > gpurun_out/p4_plain.log 2>&1
OKG_PIPE=1 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_tiled_p" -s 3 -c 1 -o gpurun_out/p4_resid2d python tools/kbench.py 2 2048 20 1 > gpurun_out/p4_ncu.log 2>&1; echo "ncu rc=$?"
OKG_PIPE=1 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_tiled_p" -s 3 -c 1 -o gpurun_out/p4_resid3d python tools/kbench.py 3 128 20 1 > gpurun_out/p4_ncu3.log 2>&1; echo "ncu rc=$?"
