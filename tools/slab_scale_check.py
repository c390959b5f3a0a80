"""Multi-slab parity at the size of BASELINE configs[4]'s weak ladder, on ONE GPU.

The 2-GPU rung of the ladder is 512^3 (135 M vertices, bench.py WEAK_N); no 2-GPU box is
available, but the thread transport runs several slabs on one device (okg_params.nslabs), and
512^3 fits one B200 (~105 GB).  This script runs the first timesteps of 512^3 once as one slab
and once as S slabs (same device, ghost-plane exchanges, replicated coarse levels, rank-ordered
reductions), and compares Newton/GMRES counts and the fields (direct relative l2).  Timing of
the S-slab run is NOT a scaling number: the slabs share the GPU.
usage: python tools/slab_scale_check.py [N=512] [SLABS=2] [STEPS=2]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_04570_b200 as okg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = okg.SolverConfig(dim=3, n=n, m=0.0, eps=0.02, dt=0.02 ** 2, gmres_tol=1e-10, gmres_restart=30,
                       min_coarse_size=17576, max_dofs=1 << 40)
N = cfg.num_vertices()
u0 = okg.seeded_ic(N, 2, 0.0)
out = {}
for slabs in (1, S):
    t0 = time.time()
    ctx = okg.SchurContext(cfg, nslabs=slabs)
    setup = time.time() - t0
    ctx.set_state(okg.State(u0, np.zeros(N)))
    counts, secs = [], []
    for _ in range(steps):
        t1 = time.time()
        st = ctx.step_resident()
        secs.append(time.time() - t1)
        counts.append((st.newton_iters, list(st.gmres_iters), bool(st.converged)))
    s = ctx.get_state()
    out[slabs] = dict(counts=counts, u=s.u, w=s.w, setup=setup, secs=secs, levels=ctx.level_sizes,
                      rep_level=ctx.rep_level, planes=ctx.slab_planes, bytes=ctx.device_bytes)
    ctx.close()
a, b = out[1], out[S]
res = {"n": n, "vertices": N, "slabs": S, "steps": steps, "levels": a["levels"], "rep_level": b["rep_level"],
       "slab_planes": b["planes"], "counts_1": a["counts"], "counts_S": b["counts"],
       "rel_u": float(np.linalg.norm(b["u"] - a["u"]) / np.linalg.norm(a["u"])),
       "rel_w": float(np.linalg.norm(b["w"] - a["w"]) / np.linalg.norm(a["w"])),
       "device_GB_1": a["bytes"] / 1e9, "device_GB_S": b["bytes"] / 1e9,
       "step_s_1": a["secs"], "step_s_S_shared_gpu": b["secs"], "setup_s": [a["setup"], b["setup"]]}
print(json.dumps(res))
assert a["counts"] == b["counts"], "iteration counts differ between 1 and S slabs"
assert res["rel_u"] <= 1e-10 and res["rel_w"] <= 1e-10
