"""Pin the oracle (CPU, no GPU): the plain-C restatement must reproduce the
reference bit-for-bit -- against the golden vectors generated from the
reference itself (tests/golden/make_golden.py) and, when oracle/_ref is built,
against the reference live -- and must satisfy the reference tests' own
known-answer checks (test_assembly.cpp, test_precond.cpp, test_multigrid.cpp,
test_model.cpp)."""
import numpy as np
import pytest

import pyoracle as po
from conftest import golden_cases, golden_params, load_golden

OPS = [("M", po.M), ("K", po.K), ("A", po.A), ("VCYCLE", po.VCYCLE), ("SHAT_INV", po.SHAT_INV),
       ("CHEB_M", po.CHEB_M), ("CHEB_A", po.CHEB_A), ("ME", po.ME), ("C", po.C_OP), ("SCHUR", po.SCHUR),
       ("SCHUR_TILDE_INV", po.SCHUR_TILDE_INV), ("S_INV_APPROX", po.S_INV_APPROX)]


@pytest.mark.parametrize("case", golden_cases())
def test_port_matches_reference_golden_bitwise(port_lib, case):
    g = load_golden(case)
    o = po.Oracle(golden_params(g, "port"), "port")
    assert [o.level_size(l) for l in range(o.levels)] == g["levels"].tolist()
    sc = o.scalars()
    got = np.array([sc[k] for k in ("c", "sqrt_c", "a_coeff", "dt_theta", "lambda_lo", "lambda_hi", "eps_sqrt_c")])
    assert np.array_equal(got, g["scalars"])
    assert np.array_equal(o.load_vector(), g["load"])
    o.set_linearization(g["u_lin"])
    for key, kind in OPS:
        assert np.array_equal(o.apply(kind, g["x"]), g["out_" + key]), key
    assert np.array_equal(o.apply(po.BLOCK, g["x2"]), g["out_BLOCK"])
    assert np.array_equal(o.apply(po.JACOBIAN, g["x2"]), g["out_JACOBIAN"])
    assert np.array_equal(o.apply(po.NONLINEAR, g["u_lin"]), g["out_NONLINEAR"])
    for l in range(o.levels):
        assert np.array_equal(o.apply(po.SHAT, g[f"xs_{l}"], level=l), g[f"out_SHAT_{l}"])
        if l + 1 < o.levels:
            assert np.array_equal(o.apply(po.PROLONG, g[f"xc_{l}"], level=l), g[f"out_PROLONG_{l}"])
            assert np.array_equal(o.apply(po.RESTRICT, g[f"xs_{l}"], level=l), g[f"out_RESTRICT_{l}"])
    assert np.array_equal(o.apply(po.COARSE_SOLVE, g["x_coarse"]), g["out_COARSE_SOLVE"])
    r = o.gmres(g["gmres_b"], 1e-10, 200, 30)
    assert r["iterations"] == int(g["gmres_iters"])
    assert np.array_equal(r["x"], g["gmres_x"])
    N = int(g["N"])
    r1, r2 = o.residual(g["u_lin"], g["res_wn"], po.seeded_ic(N, int(g["seed"]), float(g["m"]), "port"),
                        np.zeros(N))
    assert np.array_equal(r1, g["res_r1"]) and np.array_equal(r2, g["res_r2"])
    u, w = po.seeded_ic(N, int(g["seed"]), float(g["m"]), "port"), np.zeros(N)
    for s in range(2):
        u, w, st = o.newton_solve(u, w)
        assert st.newton_iters == int(g[f"newton{s}_iters"])
        assert st.gmres_iters == g[f"newton{s}_gmres"].tolist()
        assert np.array_equal(u, g[f"newton{s}_u"]) and np.array_equal(w, g[f"newton{s}_w"])


@pytest.mark.skipif(not po.available("ref"), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("dim,n,m", [(2, 12, 0.3), (3, 6, -0.2), (2, 40, 0.0)])
def test_port_matches_reference_live(port_lib, dim, n, m):
    res = {}
    for kind in ("ref", "port"):
        o = po.Oracle(po.baseline_params(dim, n, m=m, kind=kind, min_coarse_size=30), kind)
        u0 = po.seeded_ic(o.n, 5, m, kind)
        res[kind] = o.newton_solve(u0, np.zeros(o.n)), o.scalars()
    (ua, wa, sa), sca = res["ref"]
    (ub, wb, sb), scb = res["port"]
    assert sca == scb
    assert sa.gmres_iters == sb.gmres_iters
    assert np.array_equal(ua, ub) and np.array_equal(wa, wb)


@pytest.mark.parametrize("dim,n", [(2, 1), (2, 4), (3, 1), (3, 3)])
def test_mesh_ref_port(port_lib, dim, n):
    v, c = po.mesh(dim, n, "port")
    s = n + 1
    assert v.shape == (s ** dim, dim)
    assert c.shape == ((2 * n * n if dim == 2 else 6 * n ** 3), dim + 1)
    if po.available("ref"):
        v2, c2 = po.mesh(dim, n, "ref")
        assert np.array_equal(v, v2) and np.array_equal(c, c2)


def test_compute_c_kats(port_lib):
    # test_precond.cpp:105-108
    o = po.Oracle(po.default_params("port", dim=2, n=4, dt=0.0004, theta=0.5, sigma=100.0), "port")
    assert abs(o.scalars()["c"] - 0.00019607843137254902) <= 1e-15 * 0.00019607843137254902
    assert o.scalars()["a_coeff"] == 1.02
    o = po.Oracle(po.default_params("port", dim=2, n=4, dt=0.0001, theta=0.5, sigma=100.0), "port")
    assert abs(o.scalars()["c"] - 4.975124378109453e-05) <= 1e-15 * 4.975124378109453e-05


def dense(o, kind, n):
    return np.array([o.apply(kind, e) for e in np.eye(n)]).T


def test_mass_and_stiffness_kats(port_lib):
    # test_assembly.cpp:73-135 on the once-split square and a 6x6 grid
    o = po.Oracle(po.default_params("port", dim=2, n=1, min_coarse_size=1), "port")
    M = dense(o, po.M, 4)
    assert np.isclose(M[0, 0], 1 / 6) and np.isclose(M[1, 1], 1 / 12) and np.isclose(M[0, 1], 1 / 24)
    for dim, n in [(2, 6), (3, 3)]:
        o = po.Oracle(po.default_params("port", dim=dim, n=n, min_coarse_size=1000), "port")
        N = o.n
        M = dense(o, po.M, N)
        K = dense(o, po.K, N)
        assert abs(M.sum() - 1.0) <= 1e-12
        assert np.allclose(M.sum(axis=1), o.load_vector(), atol=1e-14)
        assert np.abs(K @ np.ones(N)).max() <= 1e-13
        xcoord = po.mesh(dim, n, "port")[0][:, 0]
        assert abs(xcoord @ K @ xcoord - 1.0) <= 1e-12
        # M_E(0) = -M, M_E(1) = 2M  (test_assembly.cpp:147-166)
        o.set_linearization(np.zeros(N))
        assert np.allclose(dense(o, po.ME, N), -M, atol=1e-15)
        o.set_linearization(np.ones(N))
        assert np.allclose(dense(o, po.ME, N), 2 * M, atol=1e-15)
        # N(0) = N(+-1) = 0 (test_assembly.cpp:187-194)
        for c in (0.0, 1.0, -1.0):
            assert np.abs(o.apply(po.NONLINEAR, np.full(N, c))).max() <= 1e-15


def test_hierarchy_kat(port_lib):
    # test_multigrid.cpp:34-44: 64-grid, min 100 -> 65^2, 33^2, 17^2, 9^2
    o = po.Oracle(po.default_params("port", dim=2, n=64, min_coarse_size=100), "port")
    assert [o.level_size(l) for l in range(o.levels)] == [65 * 65, 33 * 33, 17 * 17, 9 * 9]
    g = np.load(__import__("os").path.join(__import__("conftest").GOLDEN, "hierarchy64.npz"))
    assert g["levels"].tolist() == [65 * 65, 33 * 33, 17 * 17, 9 * 9]


def test_config_error_odd_grid(port_lib):
    # test_multigrid.cpp:196-202 / SURVEY 6: coarsest too large for the dense solve
    with pytest.raises(po.OracleError) as e:
        po.Oracle(po.default_params("port", dim=2, n=45), "port")
    assert e.value.kind == "ConfigError"


def test_baseline_c1_counts(port_lib):
    # C1 = 2D 64^2, seed 0 -> 1 Newton, 13 GMRES
    o = po.Oracle(po.baseline_params(2, 64, kind="port"), "port")
    u, w, st = o.newton_solve(po.seeded_ic(o.n, 0, 0.0, "port"), np.zeros(o.n))
    assert st.newton_iters == 1 and st.gmres_iters == [13] and st.converged


def test_fixed_point_zero_newton_cost(port_lib):
    # test_model.cpp:86-109
    o = po.Oracle(po.default_params("port", dim=2, n=8), "port")
    u = np.full(o.n, 0.4)
    un, wn, st = o.newton_solve(u, np.full(o.n, 0.4 ** 3 - 0.4))
    assert st.newton_iters == 0 and st.converged and np.array_equal(un, u)


def test_mass_identity(port_lib):
    # test_model.cpp:111-142: 1^T R1 identity
    p = po.default_params("port", dim=2, n=8)
    o = po.Oracle(p, "port")
    rng = np.random.default_rng(2024)
    a_u, a_w, b_u, b_w = (rng.uniform(-1, 1, o.n) for _ in range(4))
    r1, _ = o.residual(a_u, a_w, b_u, b_w)
    b = o.load_vector()
    vol = b.sum()
    mn, mo = b @ a_u, b @ b_u
    rhs = (mn - mo) + p.dt * p.sigma * (p.theta * (mn - p.m * vol) + (1 - p.theta) * (mo - p.m * vol))
    assert abs(r1.sum() - rhs) <= 1e-12


# ---- diagnostics and initial state ---------------------------------------
@pytest.mark.parametrize("case", golden_cases())
def test_port_diagnostics_match_reference_golden_bitwise(port_lib, case):
    """initial_state / total_mass / integrate_double_well / energy of the port vs the
    reference's own outputs (model.hpp:46-114, assembly.hpp:220-245)."""
    g = load_golden(case)
    o = po.Oracle(golden_params(g, "port"), "port")
    u0, w0, its = o.initial_state()
    assert np.array_equal(u0, g["init_u"]) and np.array_equal(w0, g["init_w"])
    assert its > 0
    u1, w1, st = o.newton_solve(u0, w0)
    assert np.array_equal(u1, g["init_step_u"]) and np.array_equal(w1, g["init_step_w"])
    for tag, uu in (("u0", u0), ("u1", u1)):
        assert o.total_mass(uu) == float(g[f"mass_{tag}"])
        assert o.double_well(uu) == float(g[f"well_{tag}"])
        assert o.energy(uu)[0] == float(g[f"energy_{tag}"])


@pytest.mark.skipif(not po.available("ref"), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("dim,n,m,sigma", [(2, 24, 0.2, 100.0), (3, 6, -0.1, 100.0), (2, 16, 0.0, 0.0)])
def test_port_diagnostics_match_reference_live(port_lib, dim, n, m, sigma):
    res = {}
    for kind in ("ref", "port"):
        o = po.Oracle(po.baseline_params(dim, n, m=m, kind=kind, sigma=sigma), kind)
        u0, w0, _ = o.initial_state()
        res[kind] = (u0, w0, o.total_mass(u0), o.double_well(u0), o.energy(u0)[0])
    for a, b in zip(res["ref"], res["port"]):
        assert np.array_equal(np.asarray(a), np.asarray(b))


def test_diagnostics_kats(port_lib):
    o = po.Oracle(po.baseline_params(2, 32, m=0.25, kind="port"), "port")
    u0, w0, _ = o.initial_state()
    # the cosine bump integrates to zero: b^T u0 = m (unit box)
    assert abs(o.total_mass(u0) - 0.25) < 1e-14
    # double well of a constant field c: (1 - c^2)^2
    assert abs(o.double_well(np.full(o.n, 0.5)) - 0.5625) < 1e-14
    # w0 solves M w0 = eps^2 K u0 + N(u0) to rtol 1e-12 (model.hpp:101-107)
    rhs = o.params.eps ** 2 * o.apply(po.K, u0) + o.apply(po.NONLINEAR, u0)
    assert np.linalg.norm(o.apply(po.M, w0) - rhs) <= 1e-11 * np.linalg.norm(rhs)
    # energy needs a mean-consistent field (model.hpp:68-73)
    with pytest.raises(po.OracleError, match="InconsistentState"):
        o.energy(po.seeded_ic(o.n, 1, 0.25, "port"))
