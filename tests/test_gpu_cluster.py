"""Cluster V-cycle (okg_params.mg_cluster, okg_cluster.cuh).

The latency-bound levels above the collapsed bottom run as one 16-CTA
thread-block cluster with the levels in distributed shared memory.  Every vertex
uses the unfused kernels' expressions in the same order, and the collapsed
bottom reproduces k_coarse_sym + k_coarse_sym_sum, so the cycle must be
bit-identical to the multi-launch path (mg_cluster=-1), and so must everything
built on it (multigrid.hpp:97-149, precond.hpp:199-271).  Opt-in: measured slower
than the PDL-chained level kernels.
"""
import numpy as np
import pytest

import paper_1603_04570_b200 as okg
from paper_1603_04570_b200 import _lib

pytestmark = pytest.mark.gpu

# (dim, n, mg_cluster knob, expected first cluster level n)
CASES = [(3, 32, 40000, 16), (3, 64, 40000, 32), (3, 128, 40000, 32), (3, 128, 5000, 16),
         (2, 128, 17000, 64), (2, 256, 17000, 128), (2, 512, 70000, 256), (2, 2048, 17000, 128)]


@pytest.mark.parametrize("dim,n,knob,n0", CASES)
def test_cluster_cycle_bit_identical(dim, n, knob, n0):
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
    on = okg.SchurContext(cfg, mg_cluster=knob)
    off = okg.SchurContext(cfg, mg_cluster=-1)
    assert off.mc_start == -1
    assert on.mc_start > 0 and on.info.level_n[on.mc_start] == n0
    assert on.collapse_level == off.collapse_level > on.mc_start
    rng = np.random.default_rng(n + knob)
    x = rng.uniform(-1, 1, on.n)
    for kind in (_lib.OP_VCYCLE, _lib.OP_SHAT_INV, _lib.OP_SCHUR_TILDE_INV):
        a, b = on.apply(kind, x), off.apply(kind, x)
        assert np.array_equal(a, b), (kind, np.max(np.abs(a - b)))
    # the level the cluster starts on, as a V-cycle of its own (level argument)
    xs = rng.uniform(-1, 1, int(on.level_sizes[on.mc_start]))
    assert np.array_equal(on.apply(_lib.OP_VCYCLE, xs, on.mc_start), off.apply(_lib.OP_VCYCLE, xs, on.mc_start))
    # repeated launches give the same bits
    assert np.array_equal(on.apply(_lib.OP_VCYCLE, x), on.apply(_lib.OP_VCYCLE, x))
    on.close()
    off.close()


@pytest.mark.parametrize("dim,n", [(3, 64), (2, 256)])
def test_cluster_newton_step_bit_identical(dim, n):
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
    mesh = okg.build_mesh(dim, n, False)
    res = []
    for knob in (40000, -1):
        ctx = okg.SchurContext(cfg, mg_cluster=knob)
        u0 = okg.seeded_ic(ctx.n, 2, 0.0)
        res.append(okg.newton_solve(okg.State(u0, np.zeros(ctx.n)), mesh, ctx))
        ctx.close()
    assert res[0][1].gmres_iters == res[1][1].gmres_iters
    assert np.array_equal(res[0][0].u, res[1][0].u) and np.array_equal(res[0][0].w, res[1][0].w)


def test_no_cluster_by_default_without_collapse_or_on_slabs():
    cfg = okg.SolverConfig(dim=3, n=64, m=0.0, dt=4e-4)
    for kw in (dict(), dict(mg_collapse=-1, mg_cluster=40000), dict(nslabs=2, mg_cluster=40000),
               dict(mg_cluster=-1)):
        ctx = okg.SchurContext(cfg, **kw)
        assert ctx.mc_start == -1, kw
        ctx.close()
    ctx = okg.SchurContext(okg.SolverConfig(dim=3, n=64, m=0.0, dt=4e-4, mg_pre=1, mg_post=1), mg_cluster=40000)
    assert ctx.mc_start == -1
    ctx.close()
