"""SSOR-Chebyshev (cheby_precond = ssor) on the GPU: bound agreement with the oracle
and the cost of a full-size Newton step.  usage: python tools/ssor_probe.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_1603_04570_b200 as okg  # noqa: E402
import pyoracle as po  # noqa: E402

for dim, n in ((2, 16), (2, 64), (3, 8), (3, 16)):
    ctx = okg.SchurContext(okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, cheby_iters=1, cheby_precond="ssor"))
    sc = po.Oracle(po.baseline_params(dim, n, kind="port", dt=4e-4, cheby_iters=1, cheby_ssor=1), "port").scalars()
    print(dim, n, "bounds bitwise:", ctx.lambda_lo == sc["lambda_lo"], ctx.lambda_hi == sc["lambda_hi"])
    ctx.close()
for dim, n in ((3, 128), (2, 1024)):
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, eps=0.02, dt=0.02 ** 2, gmres_tol=1e-10, gmres_restart=30,
                           cheby_precond="ssor")
    t0 = time.time()
    ctx = okg.SchurContext(cfg)
    setup = time.time() - t0
    ctx.set_state(okg.State(okg.seeded_ic(ctx.n, 2, 0.0), np.zeros(ctx.n)))
    s = ctx.step_resident()
    print(f"{dim}D n={n} ssor: setup {setup:.2f} s, step {s.seconds * 1e3:.1f} ms, newton {s.newton_iters}, "
          f"gmres {s.gmres_iters}, converged {s.converged}")
    ctx.close()
