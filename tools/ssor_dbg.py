import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, pyoracle as po, paper_1603_04570_b200 as okg
from paper_1603_04570_b200 import _lib
for dim, n in ((2, 16), (2, 32), (2, 48), (2, 64), (3, 8), (3, 24)):
    ctx = okg.SchurContext(okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, cheby_precond="ssor"))
    o = po.Oracle(po.baseline_params(dim, n, kind="port", dt=4e-4, cheby_ssor=1), "port")
    b = np.random.default_rng(n).uniform(-1, 1, ctx.n)
    a, r = ctx.apply(_lib.OP_SSOR_M, b), o.apply(po.SSOR_M, b)
    bad = np.nonzero(a != r)[0]
    print(dim, n, len(bad), bad[:8], (np.abs(a - r).max() / np.abs(r).max()) if len(bad) else 0)
