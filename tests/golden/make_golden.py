"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libokref.so,
the unmodified okflow headers compiled by oracle/Makefile).  Run in a container
where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

Each case stores its seeded inputs and the reference's outputs for every
operator on the Newton-solve path, one GMRES solve, two Newton timesteps, and
 initial_state, total_mass, integrate_double_well and energy
(BASELINE.json settings: sigma=100, theta=.5, dt=eps^2, GMRES(30) rtol 1e-10,
newton_tol 1e-8, seeded IC of SURVEY.md 8(d), w0 = 0).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as po  # noqa: E402

CASES = [
    # name, dim, n, m, eps, seed
    ("d2n8", 2, 8, 0.0, 0.02, 0),
    ("d2n16", 2, 16, 0.1, 0.02, 1),
    ("d3n4", 3, 4, 0.0, 0.02, 2),
    ("d3n8", 3, 8, 0.0, 0.02, 2),
    # deep hierarchies down to n = 2 / n = 1 grids (min_coarse_size lowered)
    ("d2n16mg", 2, 16, 0.0, 0.02, 3, 20),
    ("d3n8mg", 3, 8, 0.0, 0.02, 4, 10),
    # non-default eps / mean
    ("d2n32e01", 2, 32, 0.1, 0.01, 1),
    # cheby_precond = ssor (krylov.hpp:322-418)
    ("d2n16ssor", 2, 16, 0.1, 0.02, 1, None, 1),
    ("d3n8ssor", 3, 8, 0.0, 0.02, 2, None, 1),
    ("d2n16mgssor", 2, 16, 0.0, 0.02, 3, 20, 1),
    # coarsest level above the 2000-unknown dense default (46^2 = 2116, min_coarse_size
    # raised so the reference admits it, multigrid.hpp:67-71): the device-factorised
    # coarse inverse of the 400^3 / 800^3 hierarchies (26^3 = 17,576)
    ("d2n90big", 2, 90, 0.0, 0.02, 5, 2116),
]

OPS = [("M", po.M), ("K", po.K), ("A", po.A), ("VCYCLE", po.VCYCLE), ("SHAT_INV", po.SHAT_INV),
       ("CHEB_M", po.CHEB_M), ("CHEB_A", po.CHEB_A), ("ME", po.ME), ("C", po.C_OP), ("SCHUR", po.SCHUR),
       ("SCHUR_TILDE_INV", po.SCHUR_TILDE_INV), ("S_INV_APPROX", po.S_INV_APPROX)]


def make(name, dim, n, m, eps, seed, min_coarse=None, ssor=0):
    kw = {} if min_coarse is None else {"min_coarse_size": min_coarse}
    kw["cheby_ssor"] = ssor
    p = po.baseline_params(dim, n, eps=eps, m=m, kind="ref", **kw)
    o = po.Oracle(p, "ref")
    N = o.n
    rng = np.random.default_rng(1000 + dim * 100 + n)
    out = {"dim": dim, "n": n, "m": m, "eps": eps, "seed": seed, "N": N,
           "min_coarse": p.min_coarse_size, "ssor": ssor,
           "levels": np.array([o.level_size(l) for l in range(o.levels)])}
    sc = o.scalars()
    out["scalars"] = np.array([sc[k] for k in ("c", "sqrt_c", "a_coeff", "dt_theta", "lambda_lo",
                                                "lambda_hi", "eps_sqrt_c")])
    out["load"] = o.load_vector()
    x = rng.uniform(-1, 1, N)
    x2 = rng.uniform(-1, 1, 2 * N)
    u_lin = po.seeded_ic(N, seed, m) + 0.3 * rng.uniform(-1, 1, N)
    out["x"], out["x2"], out["u_lin"] = x, x2, u_lin
    o.set_linearization(u_lin)
    for key, kind in OPS:
        out["out_" + key] = o.apply(kind, x)
    out["out_BLOCK"] = o.apply(po.BLOCK, x2)
    out["out_JACOBIAN"] = o.apply(po.JACOBIAN, x2)
    out["out_NONLINEAR"] = o.apply(po.NONLINEAR, u_lin)
    for l in range(o.levels):
        xs = rng.uniform(-1, 1, o.level_size(l))
        out[f"xs_{l}"] = xs
        out[f"out_SHAT_{l}"] = o.apply(po.SHAT, xs, level=l)
        if l + 1 < o.levels:
            xc = rng.uniform(-1, 1, o.level_size(l + 1))
            out[f"xc_{l}"] = xc
            out[f"out_PROLONG_{l}"] = o.apply(po.PROLONG, xc, level=l)
            out[f"out_RESTRICT_{l}"] = o.apply(po.RESTRICT, xs, level=l)
    xcs = rng.uniform(-1, 1, o.level_size(o.levels - 1))
    out["x_coarse"] = xcs
    out["out_COARSE_SOLVE"] = o.apply(po.COARSE_SOLVE, xcs)
    b = rng.uniform(-1, 1, 2 * N)
    out["gmres_b"] = b
    g = o.gmres(b, 1e-10, 200, 30)
    out["gmres_x"] = g["x"]
    out["gmres_iters"] = g["iterations"]
    out["gmres_final"] = g["final_residual"]
    # residual at a perturbed state
    uo = po.seeded_ic(N, seed, m)
    wo = np.zeros(N)
    wn = rng.uniform(-1, 1, N)
    r1, r2 = o.residual(u_lin, wn, uo, wo)
    out["res_wn"], out["res_r1"], out["res_r2"] = wn, r1, r2
    # two Newton timesteps from the seeded IC
    u, w = uo, wo
    for s in range(2):
        un, wn2, st = o.newton_solve(u, w)
        out[f"newton{s}_u"] = un
        out[f"newton{s}_w"] = wn2
        out[f"newton{s}_iters"] = st.newton_iters
        out[f"newton{s}_gmres"] = np.array(st.gmres_iters)
        out[f"newton{s}_res"] = st.residual_norm
        u, w = un, wn2
    # diagnostics and initial state: initial_state, then total_mass /
    # integrate_double_well / energy at u0 and at the state after one Newton step from it
    u0, w0, _ = o.initial_state()
    out["init_u"], out["init_w"] = u0, w0
    u1, w1, st = o.newton_solve(u0, w0)
    out["init_step_u"], out["init_step_w"] = u1, w1
    out["init_step_gmres"] = np.array(st.gmres_iters)
    for tag, uu in (("u0", u0), ("u1", u1)):
        out[f"mass_{tag}"] = o.total_mass(uu)
        out[f"well_{tag}"] = o.double_well(uu)
        out[f"energy_{tag}"] = o.energy(uu)[0]
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, "levels", out["levels"], "gmres", out["gmres_iters"],
          "newton", [out["newton0_gmres"].tolist(), out["newton1_gmres"].tolist()])


if __name__ == "__main__":
    if not po.available("ref"):
        sys.exit("oracle/_ref/libokref.so missing: run `make -C oracle ref` where /root/reference exists")
    only = sys.argv[1:]
    for case in CASES:
        if not only or case[0] in only:
            make(*case)
    if only:
        sys.exit(0)
    # KAT: 64-grid hierarchy with min_coarse_size=100 (test_multigrid.cpp:34-44)
    o = po.Oracle(po.baseline_params(2, 64, kind="ref", min_coarse_size=100), "ref")
    np.savez_compressed(os.path.join(HERE, "hierarchy64.npz"),
                        levels=np.array([o.level_size(l) for l in range(o.levels)]))
