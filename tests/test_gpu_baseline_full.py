"""Parity at the BASELINE.json sizes, every timestep, against the reference itself.

tests/golden/baseline/*.npz hold, per timestep, the UNMODIFIED reference's
newton_solve (/root/reference/proj/include/okflow/model.hpp:165-215, compiled by
oracle/Makefile; fixtures made by tests/golden/make_baseline_fixtures.py) on
BASELINE configs[1] (2D 128^2 .. 2048^2, 5 steps), configs[2] (2D 1024^2, four eps,
10 steps) and configs[3] (3D 128^3, 10 steps): Newton and GMRES counts, ||u||, ||w||
and 64 Rademacher projections of u and w (tests/sketch.py), plus full fields for
2D <= 256^2 (every step) and 512^2 (last step).

The GPU replays the same timesteps from the same seeded IC through the C ABI and
must match at EVERY step (north_star): Newton iterations equal, GMRES iterations
within +-1, u and w within 1e-8 relative l2 (estimated from the projections; exact
where the full field is stored).
"""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, relerr
from sketch import est_relerr, project

import paper_1603_04570_b200 as okg

pytestmark = pytest.mark.gpu

FIELD_TOL = 1e-8
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "baseline", "*.npz")))


def load(name):
    with np.load(os.path.join(GOLDEN, "baseline", name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def test_fixture_set_complete():
    """configs[1] (5 meshes), configs[2] (4 eps), configs[3] are all pinned."""
    want = {"c2_n128", "c2_n256", "c2_n512", "c2_n1024", "c2_n2048",
            "c3_e040", "c3_e020", "c3_e010", "c3_e005", "c4_3d128"}
    assert want <= set(CASES), sorted(want - set(CASES))


@pytest.mark.parametrize("name", CASES)
def test_baseline_every_step(name):
    f = load(name)
    dim, n, eps, m, seed = int(f["dim"]), int(f["n"]), float(f["eps"]), float(f["m"]), int(f["seed"])
    cfg = okg.SolverConfig(dim=dim, n=n, eps=eps, m=m, dt=eps * eps, sigma=100.0, theta=0.5,
                           newton_tol=1e-8, gmres_tol=1e-10, gmres_restart=30)
    ctx = okg.SchurContext(cfg)
    try:
        assert ctx.n == int(f["N"])
        st = okg.State(okg.seeded_ic(ctx.n, seed, m), np.zeros(ctx.n))
        mesh = okg.build_mesh(dim, n, False)
        report = []
        for k in range(int(f["steps"])):
            st, stats = okg.newton_solve(st, mesh, ctx)
            ref_g = [int(x) for x in f["gmres_iters"][k] if x >= 0]
            assert stats.converged == bool(f["converged"][k])
            assert stats.newton_iters == int(f["newton_iters"][k]), (k, stats.newton_iters, f["newton_iters"][k])
            assert all(abs(a - b) <= 1 for a, b in zip(stats.gmres_iters, ref_g)), (k, stats.gmres_iters, ref_g)
            pu, pw = project(st.u, st.w)
            eu = est_relerr(pu, f["proj_u"][k], float(f["norm_u"][k]))
            ew = est_relerr(pw, f["proj_w"][k], float(f["norm_w"][k]))
            nu = abs(np.linalg.norm(st.u) - f["norm_u"][k]) / f["norm_u"][k]
            nw = abs(np.linalg.norm(st.w) - f["norm_w"][k]) / f["norm_w"][k]
            report.append((k + 1, stats.gmres_iters, ref_g, eu, ew))
            assert eu <= FIELD_TOL and ew <= FIELD_TOL, (k, eu, ew)
            assert nu <= FIELD_TOL and nw <= FIELD_TOL, (k, nu, nw)
            if f"u{k + 1}" in f:
                assert relerr(st.u, f[f"u{k + 1}"]) <= FIELD_TOL
                assert relerr(st.w, f[f"w{k + 1}"]) <= FIELD_TOL
        print(name, report)
    finally:
        ctx.close()
