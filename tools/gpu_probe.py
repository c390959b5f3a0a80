"""Diagnostic probe: every operator of the GPU path vs the oracle on small grids,
then Newton steps and a timing at a larger size.  Test infrastructure (uses oracle/).

usage: python tools/gpu_probe.py [--big 3:64] [--kind port|ref]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as po  # noqa: E402
import paper_1603_04570_b200 as okg  # noqa: E402
from paper_1603_04570_b200 import _lib  # noqa: E402


def rel(a, b):
    d = np.linalg.norm(a - b)
    n = np.linalg.norm(b)
    return d / n if n > 0 else d


def probe(dim, n, kind, m=0.0, seed=0):
    cfg = okg.SolverConfig(dim=dim, n=n, m=m, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
    p = po.baseline_params(dim, n, m=m, kind=kind)
    o = po.Oracle(p, kind)
    ctx = okg.SchurContext(cfg)
    print(f"== {dim}D n={n}: levels gpu={ctx.level_sizes} oracle={[o.level_size(l) for l in range(o.levels)]}")
    sc = o.scalars()
    print(f"   lambda gpu=({ctx.lambda_lo:.15g},{ctx.lambda_hi:.15g}) oracle=({sc['lambda_lo']:.15g},{sc['lambda_hi']:.15g})")
    rng = np.random.default_rng(7)
    N = o.n
    x = rng.uniform(-1, 1, N)
    x2 = rng.uniform(-1, 1, 2 * N)
    u = po.seeded_ic(N, seed, m, kind) + 0.3 * rng.uniform(-1, 1, N)
    o.set_linearization(u)
    ctx.linearize(u)
    for name, kg, ko in [("M", _lib.OP_M, po.M), ("K", _lib.OP_K, po.K), ("A", _lib.OP_A, po.A),
                         ("VCYCLE", _lib.OP_VCYCLE, po.VCYCLE), ("SHAT_INV", _lib.OP_SHAT_INV, po.SHAT_INV),
                         ("CHEB_M", _lib.OP_CHEB_M, po.CHEB_M), ("CHEB_A", _lib.OP_CHEB_A, po.CHEB_A),
                         ("ME", _lib.OP_ME, po.ME), ("C", _lib.OP_C, po.C_OP), ("SCHUR", _lib.OP_SCHUR, po.SCHUR),
                         ("STINV", _lib.OP_SCHUR_TILDE_INV, po.SCHUR_TILDE_INV),
                         ("SINV", _lib.OP_S_INV_APPROX, po.S_INV_APPROX), ("NONLIN", _lib.OP_NONLINEAR, po.NONLINEAR)]:
        arg = u if name == "NONLIN" else x
        a = ctx.apply(kg, arg)
        b = o.apply(ko, arg)
        print(f"   {name:8s} rel={rel(a, b):.3e} bitwise={np.array_equal(a, b)}")
    for name, kg, ko in [("BLOCK", _lib.OP_BLOCK, po.BLOCK), ("JAC", _lib.OP_JACOBIAN, po.JACOBIAN)]:
        a = ctx.apply(kg, x2)
        b = o.apply(ko, x2)
        print(f"   {name:8s} rel={rel(a, b):.3e}")
    for l in range(o.levels):
        xs = rng.uniform(-1, 1, o.level_size(l))
        a = ctx.apply(_lib.OP_SHAT, xs, level=l)
        b = o.apply(po.SHAT, xs, level=l)
        print(f"   SHAT[{l}] rel={rel(a, b):.3e} bitwise={np.array_equal(a, b)}")
        if l + 1 < o.levels:
            xc = rng.uniform(-1, 1, o.level_size(l + 1))
            a = ctx.apply(_lib.OP_PROLONG, xc, level=l)
            b = o.apply(po.PROLONG, xc, level=l)
            print(f"   P[{l}]    rel={rel(a, b):.3e} bitwise={np.array_equal(a, b)}")
            a = ctx.apply(_lib.OP_RESTRICT, xs, level=l)
            b = o.apply(po.RESTRICT, xs, level=l)
            print(f"   PT[{l}]   rel={rel(a, b):.3e} bitwise={np.array_equal(a, b)}")
    # residual
    w = rng.uniform(-1, 1, N)
    uo = po.seeded_ic(N, seed, m, kind)
    wo = np.zeros(N)
    r1, r2 = ctx.residual(okg.State(u, w), okg.State(uo, wo))
    q1, q2 = o.residual(u, w, uo, wo)
    print(f"   RESID    rel1={rel(r1, q1):.3e} rel2={rel(r2, q2):.3e}")
    # gmres
    b = rng.uniform(-1, 1, 2 * N)
    kg = ctx.gmres(b, 1e-10, 200, 30)
    ko = o.gmres(b, 1e-10, 200, 30)
    print(f"   GMRES    it gpu={kg.iterations} oracle={ko['iterations']} x rel={rel(kg.x, ko['x']):.3e} "
          f"final gpu={kg.final_residual:.3e} oracle={ko['final_residual']:.3e}")
    ctx.clear_linearization()
    # newton
    st = okg.State(uo, wo)
    ust, wst = uo, wo
    for step in range(2):
        t0 = time.time()
        nxt, stats = okg.newton_solve(st, None or okg.build_mesh(dim, n, with_arrays=False), ctx, cfg)
        t1 = time.time()
        un, wn, ost = o.newton_solve(ust, wst)
        print(f"   NEWTON step {step}: gpu newton={stats.newton_iters} gmres={stats.gmres_iters} res={stats.residual_norm:.3e} "
              f"t={stats.seconds:.4f}s launches={stats.kernel_launches} | oracle newton={ost.newton_iters} "
              f"gmres={ost.gmres_iters} res={ost.residual_norm:.3e} t={ost.seconds:.3f}s | "
              f"u rel={rel(nxt.u, un):.3e} w rel={rel(nxt.w, wn):.3e}")
        st, ust, wst = nxt, un, wn
    ctx.close()


def timing(dim, n, steps=3, m=0.0, seed=2):
    cfg = okg.SolverConfig(dim=dim, n=n, m=m, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
    t0 = time.time()
    ctx = okg.SchurContext(cfg)
    print(f"== timing {dim}D n={n}: setup {time.time() - t0:.2f}s levels={ctx.level_sizes} "
          f"graph_nodes={ctx.graph_nodes} bytes={ctx.device_bytes / 1e9:.2f}GB "
          f"lambda=({ctx.lambda_lo:.6f},{ctx.lambda_hi:.6f})")
    N = ctx.n
    st = okg.State(okg.seeded_ic(N, seed, m), np.zeros(N))
    ctx.set_state(st)
    for k in range(steps):
        s = ctx.step_resident()
        dofs = 2 * N * s.newton_iters
        print(f"   step {k}: newton={s.newton_iters} gmres={s.gmres_iters} res={s.residual_norm:.3e} "
              f"t={s.seconds * 1e3:.2f}ms launches={s.kernel_launches} DoF/s={dofs / s.seconds:.3e}")
    ctx.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="port")
    ap.add_argument("--big", default="3:64,2:512,3:128")
    args = ap.parse_args()
    probe(2, 16, args.kind)
    probe(3, 8, args.kind)
    probe(2, 64, args.kind)
    probe(3, 16, args.kind)
    for spec in args.big.split(","):
        if spec:
            d, n = spec.split(":")
            timing(int(d), int(n))
