"""Diagnostics and initial state on the GPU against the reference.

* golden: initial_state (u0, w0), total_mass, integrate_double_well and energy at
  u0 and after one Newton step, from the reference itself (tests/golden);
* live: the oracle's CG iteration counts, error behaviour (InconsistentState for
  a non-mean-zero potential rhs);
* slabs: the same diagnostics on 2/3 slabs agree with one slab;
* full size: run_simulation on BASELINE config 4 (3D 128^3) conserves mass.

Tolerances: u0 1e-14 (device cos vs libm, <= 1 ulp), w0 and the energy 1e-10
(the CG solves stop at rtol 1e-12 / 1e-10 and sum in another order), mass and
double well 1e-12.
"""
import numpy as np
import pytest

import pyoracle as po
from conftest import golden_cases, golden_config, golden_params, load_golden, relerr

import paper_1603_04570_b200 as okg

pytestmark = pytest.mark.gpu


def rel(a, b, floor=1e-300):
    return abs(a - b) / max(abs(b), floor)


def mass_err(a, b):
    # b^T u cancels to ~0 for m = 0: measure against the size of the summands (|u| ~ 1e-2)
    return rel(a, b, 1e-2)


@pytest.fixture(scope="module", params=golden_cases())
def gctx(request):
    g = load_golden(request.param)
    ctx = okg.SchurContext(golden_config(g))
    yield g, ctx
    ctx.close()


def test_initial_state(gctx):
    g, ctx = gctx
    st, its = ctx.initial_state()
    assert relerr(st.u, g["init_u"]) <= 1e-14
    assert relerr(st.w, g["init_w"]) <= 1e-10
    assert st.t == 0.0 and st.step == 0
    o = po.Oracle(golden_params(g, "port"), "port")
    assert abs(its - o.initial_state()[2]) <= 2


def test_diagnostics(gctx):
    g, ctx = gctx
    u0 = g["init_u"]
    for tag, u in (("u0", u0), ("u1", g["init_step_u"])):
        assert mass_err(ctx.total_mass(u), float(g[f"mass_{tag}"])) <= 1e-12, tag
        assert rel(ctx.double_well(u), float(g[f"well_{tag}"])) <= 1e-12, tag
        e, its = ctx.energy(u)
        assert rel(e, float(g[f"energy_{tag}"])) <= 1e-10, tag
        assert its > 0


def test_advance_from_initial_state(gctx):
    """advance (model.hpp:218-227): Newton step + mass + energy of the new level."""
    g, ctx = gctx
    ctx.initial_state()
    s = ctx.advance_resident(True)
    assert s.converged
    assert abs(s.newton_iters - len(g["init_step_gmres"])) == 0
    assert all(abs(a - b) <= 1 for a, b in zip(s.gmres_iters, g["init_step_gmres"].tolist()))
    st = ctx.get_state()
    assert relerr(st.u, g["init_step_u"]) <= 1e-8 and relerr(st.w, g["init_step_w"]) <= 1e-8
    assert mass_err(s.mass, float(g["mass_u1"])) <= 1e-12
    assert rel(s.energy, float(g["energy_u1"])) <= 1e-9
    # the device-resident diagnostics see the same state
    assert ctx.total_mass() == s.mass


def test_energy_errors():
    cfg = okg.SolverConfig(dim=2, n=32, m=0.1, dt=4e-4)
    ctx = okg.SchurContext(cfg)
    with pytest.raises(okg.InconsistentState):
        ctx.energy(okg.seeded_ic(ctx.n, 1, 0.1))
    with pytest.raises(okg.InvalidArgument):
        ctx.energy(np.zeros(ctx.n + 1))
    ctx.close()


def test_energy_cg_iterations_match_the_reference_2d256():
    """The energy's Jacobi CG (rtol 1e-10, <= 2000 iterations) takes as many iterations
    as the reference's (493 on 2D 256^2 for the initial state)."""
    cfg = okg.SolverConfig(dim=2, n=256, m=0.0, dt=4e-4)
    ctx = okg.SchurContext(cfg)
    st, _ = ctx.initial_state()
    e, its = ctx.energy()
    o = po.Oracle(po.baseline_params(2, 256, m=0.0, kind="port"), "port")
    eo, itso = o.energy(st.u)
    assert abs(its - itso) <= max(2, itso // 50), (its, itso)
    assert rel(e, eo) <= 1e-10
    ctx.close()


def test_sigma_zero_energy_has_no_potential_solve():
    cfg = okg.SolverConfig(dim=2, n=16, m=0.0, sigma=0.0, dt=4e-4)
    ctx = okg.SchurContext(cfg)
    st, _ = ctx.initial_state()
    e, its = ctx.energy()
    o = po.Oracle(po.baseline_params(2, 16, m=0.0, sigma=0.0, kind="port"), "port")
    assert its == 0 and rel(e, o.energy(st.u)[0]) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("dim,n,S", [(2, 64, 2), (3, 16, 2), (3, 32, 3)])
def test_diagnostics_on_slabs(dim, n, S):
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.1, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
    out = []
    for ns in (1, S):
        ctx = okg.SchurContext(cfg, nslabs=ns)
        st, its = ctx.initial_state()
        e, eits = ctx.energy()
        s = ctx.advance_resident(True)
        out.append((st, its, ctx.total_mass(st.u), ctx.double_well(st.u), e, eits, s))
        ctx.close()
    a, b = out
    assert relerr(b[0].u, a[0].u) == 0.0 and relerr(b[0].w, a[0].w) <= 1e-12
    assert abs(b[1] - a[1]) <= 1
    assert mass_err(b[2], a[2]) <= 1e-12
    for k in (3, 4):
        assert rel(b[k], a[k]) <= 1e-12, k
    assert b[6].newton_iters == a[6].newton_iters and b[6].gmres_iters == a[6].gmres_iters
    assert mass_err(b[6].mass, a[6].mass) <= 1e-12 and rel(b[6].energy, a[6].energy) <= 1e-10


def test_run_simulation_small_matches_oracle():
    """run_simulation (model.hpp:243-279) vs the oracle's initial_state + Newton loop."""
    cfg = okg.SolverConfig(dim=2, n=32, m=0.1, eps=0.02, dt=4e-4, n_steps=3, gmres_tol=1e-10,
                           gmres_restart=30)
    res = okg.run_simulation(cfg)
    o = po.Oracle(po.baseline_params(2, 32, m=0.1, eps=0.02, kind="port", dt=4e-4), "port")
    u, w, _ = o.initial_state()
    assert mass_err(res.stats[0].mass, o.total_mass(u)) <= 1e-12
    assert rel(res.stats[0].energy, o.energy(u)[0]) <= 1e-10
    for k in range(1, 4):
        u, w, st = o.newton_solve(u, w)
        s = res.stats[k]
        assert s.step == k and s.newton_iters == st.newton_iters
        assert all(abs(a - b) <= 1 for a, b in zip(s.gmres_iters, st.gmres_iters))
        assert mass_err(s.mass, o.total_mass(u)) <= 1e-12
        assert rel(s.energy, o.energy(u)[0]) <= 1e-9
    assert relerr(res.final_state.u, u) <= 1e-8


def test_full_size_3d128_run_conserves_mass():
    cfg = okg.SolverConfig(dim=3, n=128, m=0.0, eps=0.02, dt=0.02 ** 2, n_steps=2, gmres_tol=1e-10,
                           gmres_restart=30, max_dofs=3_000_000)
    res = okg.run_simulation(cfg)
    masses = [s.mass for s in res.stats]
    assert all(abs(m - masses[0]) <= 1e-12 for m in masses)
    assert all(np.isfinite(s.energy) for s in res.stats)
    assert all(s.converged for s in res.stats[1:])
