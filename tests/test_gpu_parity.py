"""Parity of the sm_100a path (through the C ABI) with the reference.

* golden: every operator on the path, one GMRES solve and two Newton steps
  against outputs of the reference itself (tests/golden/*.npz);
* live: the plain-C oracle at sizes it finishes in seconds;
* full size (BASELINE configs): size-independent properties -- convergence,
  iteration counts, linearity, the 1^T R1 mass identity, determinism.

Tolerances (north_star): iteration counts within +-1, fields within 1e-8
relative l2.  Operator applies are held to 1e-12 relative (they agree to
~1e-15 in practice: only fma contraction and summation order differ), the
grid-transfer operators P and P^T bit-exactly.
"""
import numpy as np
import pytest

import pyoracle as po
from conftest import golden_cases, golden_config, golden_params, load_golden, relerr

import paper_1603_04570_b200 as okg
from paper_1603_04570_b200 import _lib

pytestmark = pytest.mark.gpu

OP_TOL = 1e-12
FIELD_TOL = 1e-8

OPS = [("M", _lib.OP_M), ("K", _lib.OP_K), ("A", _lib.OP_A), ("VCYCLE", _lib.OP_VCYCLE),
       ("SHAT_INV", _lib.OP_SHAT_INV), ("CHEB_M", _lib.OP_CHEB_M), ("CHEB_A", _lib.OP_CHEB_A),
       ("ME", _lib.OP_ME), ("C", _lib.OP_C), ("SCHUR", _lib.OP_SCHUR),
       ("SCHUR_TILDE_INV", _lib.OP_SCHUR_TILDE_INV), ("S_INV_APPROX", _lib.OP_S_INV_APPROX)]


# kernel-path modes: default choice; shared-memory tiled kernels forced on every
# level (no single-CTA tail); one-thread-per-vertex kernels + the largest tail
MODES = {"default": {}, "tiled": dict(tiled_min_n=2, tail_max_vertices=-1, mg_fuse=1),
         "tail": dict(tiled_min_n=-1, tail_max_vertices=1 << 30, pdl=False, mg_fuse=-1)}


@pytest.fixture(scope="module", params=[(c, m) for c in golden_cases() for m in MODES],
                ids=lambda p: f"{p[0]}-{p[1]}")
def golden_ctx(request):
    case, mode = request.param
    g = load_golden(case)
    ctx = okg.SchurContext(golden_config(g), **MODES[mode])
    yield g, ctx
    ctx.close()


def test_hierarchy_and_scalars(golden_ctx):
    g, ctx = golden_ctx
    assert ctx.level_sizes == g["levels"].tolist()
    c, sqrt_c, a_coeff, dt_theta, lo, hi, esc = g["scalars"]
    assert ctx.c == c and ctx.sqrt_c == sqrt_c and ctx.a_coeff == a_coeff and ctx.dt_theta == dt_theta
    assert ctx.eps_sqrt_c == esc
    # Lanczos bounds from the same mt19937(1234) start vector; only dot-product order differs
    assert abs(ctx.lambda_lo - lo) <= 1e-12 * lo and abs(ctx.lambda_hi - hi) <= 1e-12 * hi


def test_operators(golden_ctx):
    g, ctx = golden_ctx
    ctx.linearize(g["u_lin"])
    for key, kind in OPS:
        assert relerr(ctx.apply(kind, g["x"]), g["out_" + key]) <= OP_TOL, key
    assert relerr(ctx.apply(_lib.OP_BLOCK, g["x2"]), g["out_BLOCK"]) <= OP_TOL
    assert relerr(ctx.apply(_lib.OP_JACOBIAN, g["x2"]), g["out_JACOBIAN"]) <= OP_TOL
    assert relerr(ctx.apply(_lib.OP_NONLINEAR, g["u_lin"]), g["out_NONLINEAR"]) <= OP_TOL
    assert relerr(ctx.apply(_lib.OP_COARSE_SOLVE, g["x_coarse"]), g["out_COARSE_SOLVE"]) <= OP_TOL
    for l in range(ctx.levels):
        assert relerr(ctx.apply(_lib.OP_SHAT, g[f"xs_{l}"], level=l), g[f"out_SHAT_{l}"]) <= OP_TOL
        if l + 1 < ctx.levels:
            assert np.array_equal(ctx.apply(_lib.OP_PROLONG, g[f"xc_{l}"], level=l), g[f"out_PROLONG_{l}"])
            assert np.array_equal(ctx.apply(_lib.OP_RESTRICT, g[f"xs_{l}"], level=l), g[f"out_RESTRICT_{l}"])
    ctx.clear_linearization()


def test_residual(golden_ctx):
    g, ctx = golden_ctx
    N = int(g["N"])
    old = okg.State(okg.seeded_ic(N, int(g["seed"]), float(g["m"])), np.zeros(N))
    r1, r2 = ctx.residual(okg.State(g["u_lin"], g["res_wn"]), old)
    assert relerr(r1, g["res_r1"]) <= OP_TOL and relerr(r2, g["res_r2"]) <= OP_TOL


def test_gmres(golden_ctx):
    g, ctx = golden_ctx
    ctx.linearize(g["u_lin"])
    r = ctx.gmres(g["gmres_b"], 1e-10, 200, 30)
    assert abs(r.iterations - int(g["gmres_iters"])) <= 1
    assert r.converged
    assert relerr(r.x, g["gmres_x"]) <= FIELD_TOL
    ctx.clear_linearization()


def test_newton_two_steps(golden_ctx):
    g, ctx = golden_ctx
    N = int(g["N"])
    mesh = okg.build_mesh(int(g["dim"]), int(g["n"]), with_arrays=False)
    st = okg.State(okg.seeded_ic(N, int(g["seed"]), float(g["m"])), np.zeros(N))
    for s in range(2):
        st, stats = okg.newton_solve(st, mesh, ctx)
        assert stats.converged
        assert abs(stats.newton_iters - int(g[f"newton{s}_iters"])) <= 1
        ref_g = g[f"newton{s}_gmres"].tolist()
        for a, b in zip(stats.gmres_iters, ref_g):
            assert abs(a - b) <= 1
        assert relerr(st.u, g[f"newton{s}_u"]) <= FIELD_TOL
        assert relerr(st.w, g[f"newton{s}_w"]) <= FIELD_TOL
        assert st.step == s + 1 and abs(st.t - (s + 1) * float(g["eps"]) ** 2) < 1e-15


@pytest.mark.parametrize("dim,n,m,seed", [(2, 64, 0.0, 0), (3, 16, 0.0, 2), (2, 128, 0.1, 1), (3, 24, -0.1, 3),
                                          (3, 32, 0.0, 2), (2, 256, 0.0, 0)])
def test_newton_live_oracle(port_lib, dim, n, m, seed):
    p = po.baseline_params(dim, n, m=m, kind="port")
    o = po.Oracle(p, "port")
    cfg = okg.SolverConfig(dim=dim, n=n, m=m, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
    ctx = okg.SchurContext(cfg)
    u0 = po.seeded_ic(o.n, seed, m, "port")
    un, wn, ost = o.newton_solve(u0, np.zeros(o.n))
    st, stats = okg.newton_solve(okg.State(u0, np.zeros(o.n)), okg.build_mesh(dim, n, False), ctx)
    assert stats.newton_iters == ost.newton_iters
    assert abs(stats.gmres_iters[0] - ost.gmres_iters[0]) <= 1
    assert relerr(st.u, un) <= FIELD_TOL and relerr(st.w, wn) <= FIELD_TOL
    assert stats.kernel_launches > 0


# ----------------------------------------------------------------------------------
# BASELINE full sizes: properties that do not need the oracle
# ----------------------------------------------------------------------------------
@pytest.mark.slow
@pytest.mark.parametrize("dim,n,seed,gm", [(2, 2048, 0, (8, 11)), (3, 128, 2, (11, 14))])
def test_full_size_newton(dim, n, seed, gm):
    # reference at these configs: 2D 2048^2 -> 1 Newton / 9 GMRES; 3D 128^3 -> 1 / 12
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
    ctx = okg.SchurContext(cfg)
    N = ctx.n
    u0 = okg.seeded_ic(N, seed, 0.0)
    st, stats = okg.newton_solve(okg.State(u0, np.zeros(N)), okg.build_mesh(dim, n, False), ctx)
    assert stats.converged and stats.newton_iters == 1
    assert gm[0] <= stats.gmres_iters[0] <= gm[1]
    assert np.all(np.isfinite(st.u)) and np.all(np.isfinite(st.w))
    # 1^T R1 mass identity at the new level (test_model.cpp:111-142)
    r1, r2 = ctx.residual(st, okg.State(u0, np.zeros(N)))
    b = ctx.apply(_lib.OP_M, np.ones(N))
    vol = b.sum()
    mn, mo = b @ st.u, b @ u0
    rhs = (mn - mo) + cfg.dt * cfg.sigma * (cfg.theta * (mn - cfg.m * vol) + (1 - cfg.theta) * (mo - cfg.m * vol))
    assert abs(r1.sum() - rhs) <= 1e-12
    assert np.sqrt(r1 @ r1 + r2 @ r2) <= 1e-8
    # determinism: a rerun from the same state is bit-identical
    st2, stats2 = okg.newton_solve(okg.State(u0, np.zeros(N)), okg.build_mesh(dim, n, False), ctx)
    assert stats2.gmres_iters == stats.gmres_iters
    assert np.array_equal(st2.u, st.u) and np.array_equal(st2.w, st.w)
    ctx.close()


@pytest.mark.slow
def test_block_preconditioner_linear_at_scale():
    cfg = okg.SolverConfig(dim=3, n=64, m=0.0, dt=4e-4)
    ctx = okg.SchurContext(cfg)
    N = ctx.n
    rng = np.random.default_rng(3)
    ctx.linearize(okg.seeded_ic(N, 2, 0.0))
    x, y = rng.uniform(-1, 1, 2 * N), rng.uniform(-1, 1, 2 * N)
    px, py = ctx.apply(_lib.OP_BLOCK, x), ctx.apply(_lib.OP_BLOCK, y)
    pz = ctx.apply(_lib.OP_BLOCK, 2.0 * x - 3.0 * y)
    assert relerr(pz, 2.0 * px - 3.0 * py) <= 1e-12
    ctx.close()


# ----------------------------------------------------------------------------------
# reference test properties (test_multigrid.cpp, test_precond.cpp, test_model.cpp)
# ----------------------------------------------------------------------------------
def test_vcycle_properties():
    cfg = okg.SolverConfig(dim=2, n=64, m=0.0, dt=4e-4)
    ctx = okg.SchurContext(cfg)
    N = ctx.n
    rng = np.random.default_rng(4007)
    assert np.abs(ctx.apply(_lib.OP_VCYCLE, np.zeros(N))).max() == 0.0  # maps zero to zero
    for _ in range(3):  # one V(2,2) halves the error in the operator norm
        y = rng.uniform(-1, 1, N)
        b = ctx.apply(_lib.OP_SHAT, y, level=0)
        e = y - ctx.apply(_lib.OP_VCYCLE, b)
        after = np.sqrt(e @ ctx.apply(_lib.OP_SHAT, e, level=0))
        before = np.sqrt(y @ b)
        assert after <= 0.5 * before
    b = rng.uniform(-1, 1, N)  # five cycles reach 1e-3
    x = ctx.apply(_lib.OP_SHAT_INV, b)
    assert np.linalg.norm(b - ctx.apply(_lib.OP_SHAT, x, level=0)) <= 1e-3 * np.linalg.norm(b)
    ctx.close()


def test_chebyshev_properties():
    cfg = okg.SolverConfig(dim=2, n=8)
    ctx = okg.SchurContext(cfg)
    N = ctx.n
    rng = np.random.default_rng(5)
    for _ in range(3):  # 10 steps give 1e-3 in the M-norm (test_precond.cpp:285-325)
        z = rng.uniform(-1, 1, N)
        x = ctx.apply(_lib.OP_CHEB_M, ctx.apply(_lib.OP_M, z))
        e = x - z
        assert np.sqrt(e @ ctx.apply(_lib.OP_M, e)) <= 1e-3 * np.sqrt(z @ ctx.apply(_lib.OP_M, z))
    a, b = rng.uniform(-1, 1, N), rng.uniform(-1, 1, N)  # linearity
    lhs = ctx.apply(_lib.OP_CHEB_A, 0.7 * a - 1.3 * b)
    rhs = 0.7 * ctx.apply(_lib.OP_CHEB_A, a) - 1.3 * ctx.apply(_lib.OP_CHEB_A, b)
    assert relerr(lhs, rhs) <= 1e-13
    ctx.close()


def test_fixed_point_zero_newton_cost():
    cfg = okg.SolverConfig(dim=2, n=8)
    ctx = okg.SchurContext(cfg)
    u = np.full(ctx.n, cfg.m)
    w = np.full(ctx.n, cfg.m ** 3 - cfg.m)
    st, stats = okg.newton_solve(okg.State(u, w), okg.build_mesh(2, 8, False), ctx)
    assert stats.newton_iters == 0 and stats.converged and stats.gmres_iters == []
    assert np.array_equal(st.u, u) and np.array_equal(st.w, w)
    assert st.step == 1 and st.t == cfg.dt
    ctx.close()


def test_jacobian_matches_residual_derivative():
    # test_model.cpp:144-195: finite-difference slope of the residual is the block operator
    cfg = okg.SolverConfig(dim=2, n=8)
    ctx = okg.SchurContext(cfg)
    N = ctx.n
    rng = np.random.default_rng(11)
    old = okg.State(cfg.m + 0.02 * rng.uniform(-1, 1, N), 0.1 * rng.uniform(-1, 1, N))
    base = okg.State(old.u.copy(), old.w.copy())
    ctx.linearize(base.u)
    vu, vw = rng.uniform(-1, 1, N), rng.uniform(-1, 1, N)
    Jv = ctx.apply(_lib.OP_JACOBIAN, np.concatenate([vu, vw]))
    r0 = np.concatenate(ctx.residual(base, old))

    def fd(tau):
        moved = okg.State(base.u + tau * vu, base.w + tau * vw)
        return np.linalg.norm((np.concatenate(ctx.residual(moved, old)) - r0) / tau - Jv)

    e4, e5, e6 = fd(1e-4), fd(1e-5), fd(1e-6)
    assert e4 <= 1e-3 * np.linalg.norm(Jv)
    assert e6 < e5 < e4
    assert 5.0 < e4 / e5 < 20.0 and 5.0 < e5 / e6 < 20.0
    ctx.close()


def test_error_behaviour():
    cfg = okg.SolverConfig(dim=2, n=8)
    ctx = okg.SchurContext(cfg)
    N = ctx.n
    with pytest.raises(okg.InconsistentState):   # Me not set (precond.hpp:211-213, 245-247, 281-283)
        ctx.apply(_lib.OP_C, np.zeros(N))
    with pytest.raises(okg.InconsistentState):
        ctx.apply(_lib.OP_JACOBIAN, np.zeros(2 * N))
    ctx.linearize(np.zeros(N))
    b = np.zeros(2 * N)
    b[3] = np.nan
    with pytest.raises(okg.InvalidArgument):      # require_finite (krylov.hpp:52)
        ctx.gmres(b, 1e-10, 10)
    r = ctx.gmres(np.zeros(2 * N), 1e-10, 10)     # zero rhs: converged at once
    assert r.converged and r.iterations == 0
    with pytest.raises(okg.InvalidArgument):
        okg.apply_block(ctx, np.zeros(N))
    ctx.close()
    with pytest.raises(okg.ConfigError):          # odd n: coarsest too large (test_multigrid.cpp:196-202)
        okg.SchurContext(okg.SolverConfig(dim=2, n=45))
    with pytest.raises(okg.InvalidArgument):
        okg.SchurContext(okg.SolverConfig(dim=2, n=8, eps=0.0))


def test_graphs_and_eager_agree():
    cfg = okg.SolverConfig(dim=3, n=16, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
    u0 = okg.seeded_ic(17 ** 3, 2, 0.0)
    res = []
    for graphs in (True, False):
        ctx = okg.SchurContext(cfg, use_graphs=graphs)
        st, stats = okg.newton_solve(okg.State(u0, np.zeros(u0.size)), okg.build_mesh(3, 16, False), ctx)
        res.append((st, stats))
        ctx.close()
    assert res[0][1].gmres_iters == res[1][1].gmres_iters
    assert np.array_equal(res[0][0].u, res[1][0].u)


def test_gmres_restart_and_budget():
    cfg = okg.SolverConfig(dim=2, n=32, m=0.0, dt=4e-4)
    ctx = okg.SchurContext(cfg)
    N = ctx.n
    ctx.linearize(okg.seeded_ic(N, 0, 0.0))
    b = np.random.default_rng(1).uniform(-1, 1, 2 * N)
    full = ctx.gmres(b, 1e-10, 200, 0)
    rs = ctx.gmres(b, 1e-10, 200, 4)             # restarted GMRES(4) still reaches the tolerance
    assert full.converged and rs.converged and rs.iterations >= full.iterations
    small = ctx.gmres(b, 1e-12, 3, 0)            # budget too small -> not converged
    assert not small.converged and small.iterations == 3
    norms = full.residual_norms                   # non-increasing without restart
    assert all(norms[i + 1] <= norms[i] * (1 + 1e-12) for i in range(len(norms) - 1))
    ctx.close()


def test_gmres_long_basis_chunked(port_lib):
    # a weak preconditioner needs > 32 basis vectors: exercises the chunked CGS2 path
    kw = dict(cheby_iters=1, mg_cycles=1, richardson_steps=1)
    p = po.baseline_params(2, 16, kind="port", **kw)
    o = po.Oracle(p, "port")
    cfg = okg.SolverConfig(dim=2, n=16, m=0.0, dt=4e-4, **kw)
    ctx = okg.SchurContext(cfg)
    u = okg.seeded_ic(ctx.n, 0, 0.0)
    ctx.linearize(u)
    o.set_linearization(u)
    b = np.random.default_rng(9).uniform(-1, 1, 2 * ctx.n)
    r = ctx.gmres(b, 1e-10, 100, 0)
    ro = o.gmres(b, 1e-10, 100, 0)
    assert ro["iterations"] > 32
    assert abs(r.iterations - ro["iterations"]) <= 1 and r.converged
    assert relerr(r.x, ro["x"]) <= FIELD_TOL
    ctx.close()


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 9, 10])
@pytest.mark.parametrize("dim,n,mode", [(2, 32, "tiled"), (3, 8, "tiled"), (2, 32, "plain"), (3, 32, "default")])
def test_chebyshev_iteration_counts(monkeypatch, port_lib, k, dim, n, mode):
    """chebyshev_semi_iteration (krylov.hpp:158-202) for every parity of the iteration count: the
    tiled path updates x every other step ((x + d_k) + d_{k+1}) and forms the start vector in the
    first step's staging transform (L_CHEB0) -- both must keep the oracle's values, and the fused
    start vector the bits of the separate kernel."""
    modes = dict(MODES, plain=dict(tiled_min_n=-1, mg_fuse=-1))
    p = po.baseline_params(dim, n, kind="port", cheby_iters=k)
    o = po.Oracle(p, "port")
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, cheby_iters=k)
    x = np.random.default_rng(10 * k + n).uniform(-1, 1, (n + 1) ** dim)
    outs = []
    for fuse0 in ("1", "0"):
        monkeypatch.setenv("OKG_CHEB0", fuse0)
        ctx = okg.SchurContext(cfg, **modes[mode])
        outs.append([ctx.apply(kind, x) for kind in (_lib.OP_CHEB_M, _lib.OP_CHEB_A)])
        ctx.close()
    for kind, y in zip((po.CHEB_M, po.CHEB_A), outs[0]):
        assert relerr(y, o.apply(kind, x)) <= OP_TOL
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


KNOBS = [dict(cheby_iters=1, mg_cycles=1, richardson_steps=1), dict(mg_pre=1, mg_post=0),
         dict(mg_pre=3, mg_post=1), dict(mg_pre=0, mg_post=2), dict(mg_omega=0.8, richardson_steps=3),
         dict(cheby_iters=4, mg_cycles=2)]


@pytest.mark.parametrize("kw", KNOBS, ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()))
@pytest.mark.parametrize("dim,n,mode", [(2, 32, "default"), (2, 32, "tiled"), (3, 8, "tiled"), (3, 8, "tail")])
def test_solver_knobs_match_oracle(port_lib, kw, dim, n, mode):
    p = po.baseline_params(dim, n, kind="port", min_coarse_size=10, **kw)
    o = po.Oracle(p, "port")
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, min_coarse_size=10, **kw)
    ctx = okg.SchurContext(cfg, **MODES[mode])
    assert ctx.level_sizes == [o.level_size(l) for l in range(o.levels)]
    u = okg.seeded_ic(ctx.n, 1, 0.0) + 0.2 * np.random.default_rng(1).uniform(-1, 1, ctx.n)
    ctx.linearize(u)
    o.set_linearization(u)
    x2 = np.random.default_rng(2).uniform(-1, 1, 2 * ctx.n)
    assert relerr(ctx.apply(_lib.OP_BLOCK, x2), o.apply(po.BLOCK, x2)) <= OP_TOL
    b = np.random.default_rng(3).uniform(-1, 1, 2 * ctx.n)
    r = ctx.gmres(b, 1e-10, 100, 30)
    ro = o.gmres(b, 1e-10, 100, 30)
    assert abs(r.iterations - ro["iterations"]) <= 1 and r.converged == ro["converged"]
    assert relerr(r.x, ro["x"]) <= FIELD_TOL
    ctx.close()


@pytest.mark.parametrize("dim,n", [(3, 64), (3, 48), (3, 72), (3, 40), (2, 512), (2, 320), (2, 136)])
def test_wide_staging_bit_identical(monkeypatch, dim, n):
    """k_tiled's 16-byte staging (rows fetched from their address rounded down to 16 bytes, the
    row parity folded into the tap addresses) against the 8-byte staging: every tiled operator
    and a Newton step have the same bits -- on grids whose tiles are cut by the box (40, 48,
    72, 136, 320), for both halves of a stacked vector (the w half of [u; w] starts 8 bytes into a
    16-byte chunk when N is odd) and on every tiled level (tiled_min_n=2: thin tiles too)."""
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
    rng = np.random.default_rng(n)
    x = rng.uniform(-1, 1, (n + 1) ** dim)
    x2 = rng.uniform(-1, 1, 2 * (n + 1) ** dim)
    u0 = okg.seeded_ic((n + 1) ** dim, 1, 0.0)
    outs = []
    for wide, extra in (("0", {}), ("", {}), ("", dict(tiled_min_n=2, mg_fuse=-1, tail_max_vertices=-1))):
        if wide:
            monkeypatch.setenv("OKG_WIDE", wide)
        else:
            monkeypatch.delenv("OKG_WIDE", raising=False)
        ctx = okg.SchurContext(cfg, **extra)
        ctx.linearize(u0)
        res = [ctx.apply(k, x) for k in (_lib.OP_M, _lib.OP_K, _lib.OP_SHAT, _lib.OP_VCYCLE, _lib.OP_SHAT_INV,
                                         _lib.OP_CHEB_M, _lib.OP_CHEB_A, _lib.OP_SCHUR_TILDE_INV)]
        res += [ctx.apply(k, x2) for k in (_lib.OP_BLOCK, _lib.OP_JACOBIAN)]
        ctx.clear_linearization()
        st, stats = okg.newton_solve(okg.State(u0, np.zeros_like(u0)), okg.build_mesh(dim, n, False), ctx)
        res += [st.u, st.w]
        outs.append((res, stats.gmres_iters))
        ctx.close()
    for other in outs[1:2]:  # same kernel choice, only the staging differs: same bits
        assert other[1] == outs[0][1]
        for a, b in zip(other[0], outs[0][0]):
            assert np.array_equal(a, b)
    # every level tiled (other kernels on the small levels): same iteration counts, fields to rounding
    assert outs[2][1] == outs[0][1]
    assert relerr(outs[2][0][-2], outs[0][0][-2]) <= 1e-10


@pytest.mark.parametrize("dim,n", [(2, 64), (2, 256), (3, 32), (3, 16), (3, 64)])
def test_fused_vcycle_bit_identical(dim, n):
    # okg_vcycle.cuh claims the same arithmetic per vertex as the unfused kernels
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, min_coarse_size=10)
    rng = np.random.default_rng(5)
    outs = []
    big = 1 << 30
    for mode in (dict(mg_fuse=-1, tail_max_vertices=-1), dict(mg_fuse=1, tail_max_vertices=-1),
                 dict(mg_fuse=0, tail_max_vertices=-1), dict(mg_fuse=0),
                 dict(tail_max_vertices=big, tail_cluster=16), dict(tail_max_vertices=big, tail_cluster=1),
                 dict(tail_max_vertices=big, tail_cluster=4), dict(tail_max_vertices=2000, tail_cluster=8)):
        ctx = okg.SchurContext(cfg, **mode)
        x = rng.uniform(-1, 1, ctx.n) if not outs else outs[0][0]
        outs.append((x, ctx.apply(_lib.OP_VCYCLE, x), ctx.apply(_lib.OP_SHAT_INV, x)))
        ctx.close()
    for o in outs[1:]:
        assert np.array_equal(o[1], outs[0][1]) and np.array_equal(o[2], outs[0][2])


@pytest.mark.parametrize("dim,n", [(2, 16), (2, 48), (2, 64), (3, 8), (3, 16), (3, 24)])
def test_ssor_sweeps_bit_exact(dim, n):
    """okg_ssor.cuh: the hyperplane-wavefront SSOR sweeps reproduce the reference's
    sequential SsorSweeps(M, 1).apply_inv bit for bit (power-of-two grids); the Lanczos bounds of
    estimate_ssor_spectrum agree to rounding (dot-product order)."""
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, cheby_precond="ssor")
    ctx = okg.SchurContext(cfg)
    o = po.Oracle(po.baseline_params(dim, n, kind="port", dt=4e-4, cheby_ssor=1), "port")
    b = np.random.default_rng(n).uniform(-1, 1, ctx.n)
    got, want = ctx.apply(_lib.OP_SSOR_M, b), o.apply(po.SSOR_M, b)
    if n & (n - 1) == 0:  # power-of-two grid: the class tables are the reference's CSR rows exactly
        assert np.array_equal(got, want)
    else:  # the reference's element matrices carry coordinate rounding (i*h inexact)
        assert relerr(got, want) <= 1e-13
    sc = o.scalars()
    assert abs(ctx.lambda_lo - sc["lambda_lo"]) <= 1e-12 * sc["lambda_lo"]
    assert abs(ctx.lambda_hi - sc["lambda_hi"]) <= 1e-12 * sc["lambda_hi"]
    ctx.close()


def test_ssor_rejects_slabs():
    cfg = okg.SolverConfig(dim=2, n=64, m=0.0, dt=4e-4, cheby_precond="ssor")
    with pytest.raises(okg.ConfigError, match="ssor"):
        okg.SchurContext(cfg, nslabs=2)


@pytest.mark.parametrize("dim,n", [(2, 48), (2, 50), (2, 100), (3, 24), (3, 40)])
def test_non_power_of_two_grids(dim, n):
    """eps-study meshes (n = round(2/eps): 50, 100, ...) and other n = 2^k * odd."""
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30, max_dofs=10 ** 7)
    ctx = okg.SchurContext(cfg)
    st0 = okg.State(okg.seeded_ic(ctx.n, 1, 0.0), np.zeros(ctx.n))
    ctx.set_state(st0)
    s = ctx.step_resident()
    o = po.Oracle(po.baseline_params(dim, n, kind="port", dt=4e-4), "port")
    un, wn, ost = o.newton_solve(st0.u, st0.w)
    assert s.converged and s.newton_iters == ost.newton_iters
    assert all(abs(a - b) <= 1 for a, b in zip(s.gmres_iters, ost.gmres_iters))
    assert relerr(ctx.get_state().u, un) <= 1e-8
    ctx.close()
