"""Bit-identity check between libokg builds: python tools/ab_bits.py OUT.npz
(OKG_LIB selects the build) writes the V-cycle / Shat^-1 / block-preconditioner
outputs and one Newton step's fields for a few grids; compare two files with
python tools/ab_bits.py --cmp A.npz B.npz."""
import os
import sys

import numpy as np

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print(f"{len(a.files)} arrays, {len(bad)} differ: {bad}")
    sys.exit(1 if bad else 0)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_04570_b200 as okg  # noqa: E402
from paper_1603_04570_b200 import _lib  # noqa: E402

out = {}
for dim, n in ((3, 64), (3, 128), (2, 512), (2, 2048)):
    ctx = okg.SchurContext(okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30))
    x = np.random.default_rng(n).uniform(-1, 1, ctx.n)
    for kind in (_lib.OP_VCYCLE, _lib.OP_SHAT_INV):
        out[f"{dim}_{n}_{kind}"] = ctx.apply(kind, x)
    u0 = okg.seeded_ic(ctx.n, 2, 0.0)
    st, stats = okg.newton_solve(okg.State(u0, np.zeros(ctx.n)), okg.build_mesh(dim, n, False), ctx)
    out[f"{dim}_{n}_u"], out[f"{dim}_{n}_w"] = st.u, st.w
    ctx.close()
np.savez(sys.argv[1], **out)
print("wrote", sys.argv[1], len(out))
