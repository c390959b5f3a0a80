set -u
mkdir -p gpurun_out
export OKG_MIN_COARSE=17576
for P in 1 0; do OKG_PDL=$P timeout 300 python tools/kbench.py 3 400 20 > gpurun_out/r16_kb400_pdl$P.log 2>&1; done
for f in gpurun_out/r16_kb*; do echo $f; cat $f; done
