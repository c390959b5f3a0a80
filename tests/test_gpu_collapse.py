"""Collapsed bottom of the V-cycle (okg_params.mg_collapse).

Below some coarse level l_c the V(2,2) cycle -- damped-Jacobi sweeps, P^T, P and
the exact coarse solve -- is a fixed linear map of the level-l_c right-hand side,
symmetric because the post-smoother is the pre-smoother's adjoint
(multigrid.hpp:97-117).  The context forms it once at setup from the existing
kernels (columns = the cycle applied to unit vectors) and applies it as one
packed-symmetric matvec.  It must agree with the recursive cycle to rounding, and
the solver must take the same iterations to the same fields.
"""
import numpy as np
import pytest

from conftest import relerr

import paper_1603_04570_b200 as okg
from paper_1603_04570_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dim,n", [(3, 32), (3, 64), (3, 128), (2, 256), (2, 512), (2, 2048)])
def test_collapse_matches_recursive_cycle(dim, n):
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
    on = okg.SchurContext(cfg)
    off = okg.SchurContext(cfg, mg_collapse=-1)
    assert off.collapse_level == -1
    assert 0 < on.collapse_level < on.levels - 1
    assert on.level_sizes[on.collapse_level] <= (1000 if dim == 3 else 1100)
    rng = np.random.default_rng(n)
    x = rng.uniform(-1, 1, on.n)
    for kind in (_lib.OP_VCYCLE, _lib.OP_SHAT_INV, _lib.OP_SCHUR_TILDE_INV):
        assert relerr(on.apply(kind, x), off.apply(kind, x)) <= 1e-13, kind
    assert np.array_equal(on.apply(_lib.OP_VCYCLE, x), on.apply(_lib.OP_VCYCLE, x))
    u0 = okg.seeded_ic(on.n, 2, 0.0)
    res = [okg.newton_solve(okg.State(u0, np.zeros(on.n)), okg.build_mesh(dim, n, False), c) for c in (on, off)]
    assert res[0][1].gmres_iters == res[1][1].gmres_iters
    assert relerr(res[0][0].u, res[1][0].u) <= 1e-10 and relerr(res[0][0].w, res[1][0].w) <= 1e-10
    on.close()
    off.close()


def test_no_collapse_without_an_eligible_level():
    # 48^3: levels 49^3, 25^3, 13^3, 7^3 -- the only level <= 1000 vertices is the coarsest
    ctx = okg.SchurContext(okg.SolverConfig(dim=3, n=48, m=0.0, dt=4e-4))
    assert ctx.collapse_level == -1
    ctx.close()


def test_collapse_only_with_symmetric_cycles():
    cfg = okg.SolverConfig(dim=3, n=32, m=0.0, dt=4e-4, mg_pre=2, mg_post=1)
    ctx = okg.SchurContext(cfg)
    assert ctx.collapse_level == -1
    ctx.close()
