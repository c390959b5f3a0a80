import sys, numpy as np
sys.path.insert(0, '.')
import paper_1603_04570_b200 as okg
from paper_1603_04570_b200 import _lib
for dim, n in [(2, 16), (3, 8)]:
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, min_coarse_size=1000)
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (n + 1) ** dim)
    out = {}
    for name, mode in [("simple", dict(mg_fuse=-1, tiled_min_n=-1)), ("tiled", dict(mg_fuse=-1, tiled_min_n=2))]:
        ctx = okg.SchurContext(cfg, **mode)
        out[name] = {k: ctx.apply(getattr(_lib, "OP_" + k), x) for k in ("M", "K", "A", "CHEB_M", "CHEB_A")}
        out[name]["SHAT0"] = ctx.apply(_lib.OP_SHAT, x, level=0)
        ctx.close()
    for k in out["simple"]:
        a, b = out["simple"][k], out["tiled"][k]
        bad = np.nonzero(a != b)[0]
        print(dim, n, k, "ndiff", len(bad), "maxdiff", np.abs(a - b).max(), "first", bad[:8])
