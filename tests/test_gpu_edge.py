"""Edge cases of the reference's path on the GPU, against the oracle:

* GMRES breakdown -> `stagnated` (krylov.hpp:117-120, 145-148): rel_tol = 0 on a
  tiny mesh exhausts the 2N-dimensional Krylov space, the Arnoldi norm collapses
  below 1e-13 of the column norm and the solve returns stagnated, not converged;
* `shat_perturb != 0` fault injection (precond.hpp:139-143): S-hat scaled by
  (1 + shat_perturb); a non-positive scale is std::invalid_argument;
* host arrays of the wrong length are std::invalid_argument before anything is
  read or written (LinearOperator::apply, operator.hpp:22-25; gmres,
  krylov.hpp:48-51; residual, model.hpp:126-127).
"""
import numpy as np
import pytest

import pyoracle as po
from conftest import relerr

import paper_1603_04570_b200 as okg
from paper_1603_04570_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dim,n,restart", [(2, 2, 0), (2, 4, 0), (3, 2, 0), (2, 4, 60)])
def test_gmres_stagnation_matches_oracle(port_lib, dim, n, restart):
    p = po.baseline_params(dim, n, kind="port")
    o = po.Oracle(p, "port")
    ctx = okg.SchurContext(okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4))
    try:
        u = okg.seeded_ic(ctx.n, 1, 0.0)
        ctx.linearize(u)
        o.set_linearization(u)
        b = np.random.default_rng(3).uniform(-1, 1, 2 * ctx.n)
        r = ctx.gmres(b, 0.0, 200, restart)
        ro = o.gmres(b, 0.0, 200, restart)
        assert ro["stagnated"] and not ro["converged"] and ro["iterations"] == 2 * ctx.n
        assert r.stagnated and not r.converged
        assert abs(r.iterations - ro["iterations"]) <= 1, (r.iterations, ro["iterations"])
        assert r.final_residual <= 1e-12 * np.linalg.norm(b)
        assert relerr(r.x, ro["x"]) <= 1e-8
    finally:
        ctx.close()


@pytest.mark.parametrize("perturb", [0.3, -0.5, 2.0])
@pytest.mark.parametrize("dim,n", [(2, 16), (3, 8)])
def test_shat_perturb_matches_oracle(port_lib, dim, n, perturb):
    p = po.baseline_params(dim, n, kind="port", shat_perturb=perturb)
    o = po.Oracle(p, "port")
    ctx = okg.SchurContext(okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30),
                           shat_perturb=perturb)
    try:
        assert ctx.eps_sqrt_c == o.scalars()["eps_sqrt_c"]
        u = okg.seeded_ic(ctx.n, 2, 0.0)
        ctx.linearize(u)
        o.set_linearization(u)
        x = np.random.default_rng(5).uniform(-1, 1, ctx.n)
        for kind, okind in [(_lib.OP_SHAT, po.SHAT), (_lib.OP_SHAT_INV, po.SHAT_INV),
                            (_lib.OP_SCHUR_TILDE_INV, po.SCHUR_TILDE_INV), (_lib.OP_S_INV_APPROX, po.S_INV_APPROX)]:
            assert relerr(ctx.apply(kind, x), o.apply(okind, x)) <= 1e-12, kind
        x2 = np.random.default_rng(6).uniform(-1, 1, 2 * ctx.n)
        assert relerr(ctx.apply(_lib.OP_BLOCK, x2), o.apply(po.BLOCK, x2)) <= 1e-12
        b = np.random.default_rng(7).uniform(-1, 1, 2 * ctx.n)
        r = ctx.gmres(b, 1e-10, 100, 30)
        ro = o.gmres(b, 1e-10, 100, 30)
        assert abs(r.iterations - ro["iterations"]) <= 1 and r.converged == ro["converged"]
        assert relerr(r.x, ro["x"]) <= 1e-8
    finally:
        ctx.close()


def test_shat_perturb_nonpositive_scale_rejected(port_lib):
    with pytest.raises(po.OracleError):
        po.Oracle(po.baseline_params(2, 8, kind="port", shat_perturb=-1.0), "port")
    with pytest.raises(okg.InvalidArgument):
        okg.SchurContext(okg.SolverConfig(dim=2, n=8, m=0.0, dt=4e-4), shat_perturb=-1.0)


def test_host_length_mismatch_raises():
    ctx = okg.SchurContext(okg.SolverConfig(dim=2, n=32, m=0.0, dt=4e-4))
    try:
        assert len(ctx.level_sizes) >= 2
        N = ctx.n
        u = okg.seeded_ic(N, 0, 0.0)
        with pytest.raises(okg.InvalidArgument):
            ctx.linearize(u[:-1])
        ctx.linearize(u)
        for kind, nin in [(_lib.OP_M, N), (_lib.OP_BLOCK, 2 * N), (_lib.OP_JACOBIAN, 2 * N),
                          (_lib.OP_SHAT, ctx.level_sizes[1])]:
            lvl = 1 if kind == _lib.OP_SHAT else 0
            with pytest.raises(okg.InvalidArgument):
                ctx.apply(kind, np.zeros(nin - 1), level=lvl)
            with pytest.raises(okg.InvalidArgument):
                ctx.apply(kind, np.zeros(nin + 7), level=lvl)
            assert ctx.apply(kind, np.ones(nin), level=lvl).size == nin
        with pytest.raises(okg.InvalidArgument):
            ctx.gmres(np.ones(2 * N - 1), 1e-10, 10)
        s = okg.State(u, np.zeros(N))
        with pytest.raises(okg.InvalidArgument):
            ctx.residual(okg.State(u[:-1], np.zeros(N - 1)), s)
        r1, r2 = ctx.residual(s, s)
        assert r1.size == N and r2.size == N
    finally:
        ctx.close()
