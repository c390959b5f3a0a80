"""BASELINE configs against the reference's own iteration counts.

The counts are the reference's newton_solve on the same seeded inputs (SURVEY.md
§6 "measured here": seeded IC of §8(d), w0 = 0, GMRES(30) rtol 1e-10,
newton_tol 1e-8, dt = eps^2, sigma = 100, theta = 0.5).  The GPU solve must take
the same number of Newton steps and the same GMRES iterations within +-1
(north star: "identical GMRES/Newton iteration counts within +-1").
"""
import numpy as np
import pytest

import paper_1603_04570_b200 as okg

pytestmark = pytest.mark.gpu

# configs[1] mesh-independence sweep (first steps; 128^2: five steps)
MESH = [(2, 128, [12, 14, 14, 14, 13]), (2, 256, [11]), (2, 512, [10]), (2, 1024, [9]), (2, 2048, [9]),
        (3, 32, [13]), (3, 64, [13]), (3, 128, [12])]
# configs[2] eps-robustness sweep at 1024^2, m = 0.1, seed 1 (first step)
EPS = [(0.04, 9), (0.02, 9), (0.01, 10), (0.005, 11)]


def run(dim, n, eps, m, seed, steps):
    cfg = okg.SolverConfig(dim=dim, n=n, eps=eps, m=m, dt=eps * eps, sigma=100.0, theta=0.5,
                           newton_tol=1e-8, gmres_tol=1e-10, gmres_restart=30)
    ctx = okg.SchurContext(cfg)
    st = okg.State(okg.seeded_ic(ctx.n, seed, m), np.zeros(ctx.n))
    mesh = okg.build_mesh(dim, n, False)
    out = []
    for _ in range(steps):
        st, stats = okg.newton_solve(st, mesh, ctx)
        assert stats.converged and stats.newton_iters == 1
        out.append(stats.gmres_iters[0])
    ctx.close()
    return out


@pytest.mark.parametrize("dim,n,ref", MESH, ids=[f"{d}d{n}" for d, n, _ in MESH])
def test_mesh_sweep_counts(dim, n, ref):
    seed = 0 if dim == 2 else 2
    got = run(dim, n, 0.02, 0.0, seed, len(ref))
    assert all(abs(a - b) <= 1 for a, b in zip(got, ref)), (got, ref)


@pytest.mark.parametrize("eps,ref", EPS)
def test_eps_sweep_counts(eps, ref):
    got = run(2, 1024, eps, 0.1, 1, 1)
    assert abs(got[0] - ref) <= 1, (got, ref)
