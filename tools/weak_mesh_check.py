"""One Newton step on each weak-scaling mesh of bench.py (WEAK_N), one slab and,
emulated on one GPU, the slab count the N-GPU run would use."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_04570_b200 as okg  # noqa: E402

cases = [(3, 160, 2), (3, 192, 4), (3, 256, 8), (2, 2944, 2), (2, 4096, 4), (2, 5888, 8)]
only = sys.argv[1:]
for dim, n, S in cases:
    if only and f"{dim}d{n}" not in only:
        continue
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, eps=0.02, dt=0.02 ** 2, gmres_tol=1e-10, gmres_restart=30,
                           max_dofs=10 ** 9)
    for ns in (1, S):
        t0 = time.time()
        ctx = okg.SchurContext(cfg, nslabs=ns)
        setup = time.time() - t0
        ctx.set_state(okg.State(okg.seeded_ic(ctx.n, 2, 0.0), np.zeros(ctx.n)))
        s = ctx.step_resident()
        print(f"{dim}D n={n} slabs={ns}: levels={ctx.level_sizes} setup {setup:.1f}s step {s.seconds*1e3:.0f} ms "
              f"newton {s.newton_iters} gmres {s.gmres_iters} conv {s.converged} MB={ctx.device_bytes/1e6:.0f}",
              flush=True)
        ctx.close()
