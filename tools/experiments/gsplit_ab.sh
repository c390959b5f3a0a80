# NOT ADOPTED (the okg_host.cu side was reverted): A/B driver of the graph-chain experiment
# head of the next GMRES iteration's graph chain launched before the host waits for the reductions
# (OKG_GRAPH_SPLIT = kernel counts where the chain is cut) against one graph per iteration ("0")
SPS=${SPS:-0 6 3 12 6,60}
for SP in $SPS; do
  OKG_GRAPH_SPLIT=$SP timeout 600 python tools/ab_bits.py gpurun_out/bits_$SP.npz > /dev/null 2>&1
  [ $SP != 0 ] && echo "bits 0 vs $SP: $(timeout 100 python tools/ab_bits.py --cmp gpurun_out/bits_0.npz gpurun_out/bits_$SP.npz 2>&1 | tail -1)"
done
rm -f gpurun_out/bits_*.npz
for rep in 1 2; do for SP in $SPS; do for WL in c4_3d128 c2_2d2048; do
  r=$(OKG_GRAPH_SPLIT=$SP timeout 300 python bench.py --workload $WL --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,2), d['gmres_iters'][:3])")
  echo "step $WL split=$SP rep$rep $r"; done; done; done
for SP in 0 6; do
  r=$(OKG_GRAPH_SPLIT=$SP timeout 600 python bench.py --workload c5_3d800 --steps 3 --no-cpu-baseline --no-kernels 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['gmres_iters'][:3])"); echo "step 400 split=$SP $r"
done
