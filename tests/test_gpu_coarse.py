"""Large coarsest level (> 2000 unknowns): the device-factorised coarse inverse.

The reference caps its dense coarse Cholesky at max(min_coarse_size, 2000)
unknowns (multigrid.hpp:52,67-71); raising min_coarse_size admits bigger ones,
which is what BASELINE config 5 needs (400^3 per-GPU slice and 800^3 coarsen to
26^3 = 17,576).  Above 2000 unknowns the context factorises the coarsest
operator on the device once (cuSOLVER potrf/potri at setup) and applies the
inverse with its own HBM-streaming kernel (k_coarse_gemv); on a split hierarchy
each slab multiplies the rows of its own coarse planes and the planes are
all-gathered.

Checked here against the oracle (the port, pinned bit-exact to the reference on
the d2n90big golden case, tests/test_oracle.py) and across slab counts.
"""
import numpy as np
import pytest

from conftest import relerr

import paper_1603_04570_b200 as okg
import pyoracle as po
from paper_1603_04570_b200 import _lib

pytestmark = pytest.mark.gpu

OP_TOL = 1e-12
FIELD_TOL = 1e-8

# (dim, n, min_coarse_size): coarsest 46^2 = 2116, 14^3 = 2744, 16^3 = 4096
CASES = [(2, 90, 2116), (3, 26, 2744), (3, 30, 4096)]


def cfg_for(dim, n, mcs, m=0.0):
    return okg.SolverConfig(dim=dim, n=n, m=m, eps=0.02, dt=4e-4, gmres_tol=1e-10, gmres_restart=30,
                            newton_tol=1e-8, min_coarse_size=mcs)


@pytest.mark.parametrize("dim,n,mcs", CASES)
def test_operators_and_newton_vs_oracle(port_lib, dim, n, mcs):
    o = po.Oracle(po.baseline_params(dim, n, kind="port", min_coarse_size=mcs), "port")
    ctx = okg.SchurContext(cfg_for(dim, n, mcs))
    assert ctx.level_sizes == [o.level_size(l) for l in range(o.levels)]
    assert ctx.level_sizes[-1] > 2000
    rng = np.random.default_rng(dim * 1000 + n)
    xc = rng.uniform(-1, 1, ctx.level_sizes[-1])
    assert relerr(ctx.apply(_lib.OP_COARSE_SOLVE, xc), o.apply(po.COARSE_SOLVE, xc)) <= OP_TOL
    x = rng.uniform(-1, 1, ctx.n)
    for kind in (po.VCYCLE, po.SHAT_INV, po.SCHUR_TILDE_INV):
        assert relerr(ctx.apply(kind, x), o.apply(kind, x)) <= OP_TOL, kind
    u0 = po.seeded_ic(o.n, 2, 0.0, "port")
    un, wn, ost = o.newton_solve(u0, np.zeros(o.n))
    st, stats = okg.newton_solve(okg.State(u0, np.zeros(o.n)), okg.build_mesh(dim, n, False), ctx)
    assert stats.newton_iters == ost.newton_iters
    assert all(abs(a - b) <= 1 for a, b in zip(stats.gmres_iters, ost.gmres_iters))
    assert relerr(st.u, un) <= FIELD_TOL and relerr(st.w, wn) <= FIELD_TOL
    ctx.close()


def test_misaligned_rhs_and_rerun_bit_identical():
    ctx = okg.SchurContext(cfg_for(3, 26, 2744))
    nc = ctx.level_sizes[-1]
    rng = np.random.default_rng(3)
    buf = rng.uniform(-1, 1, nc + 1)
    a = okg.DeviceArray.from_numpy(buf)
    y = okg.DeviceArray(nc)
    # an rhs 8 bytes off the 16-byte alignment k_coarse_gemv streams with
    ctx.apply_dev(_lib.OP_COARSE_SOLVE, okg.DeviceArray.view(a, 1, nc), y)
    ref = ctx.apply(_lib.OP_COARSE_SOLVE, buf[1:].copy())
    assert np.array_equal(y.numpy(), ref)
    assert np.array_equal(ctx.apply(_lib.OP_COARSE_SOLVE, buf[1:].copy()), ref)
    ctx.close()


@pytest.mark.parametrize("dim,n,mcs,S", [(2, 90, 2116, 2), (2, 90, 2116, 3), (3, 26, 2744, 2),
                                         (3, 30, 4096, 3)])
@pytest.mark.parametrize("split", [0, -1])
def test_slabs_split_coarse_rows(dim, n, mcs, S, split):
    cfg = cfg_for(dim, n, mcs)
    one = okg.SchurContext(cfg, coarse_split=-1)  # full rows (one slab would pack the symmetric blocks)
    many = okg.SchurContext(cfg, nslabs=S, coarse_split=split)
    assert many.rep_level == many.levels - 1  # the coarsest is the first replicated level
    nc = one.level_sizes[-1]
    assert one.coarse_rows == nc
    assert (many.coarse_rows < nc) if split == 0 else (many.coarse_rows == nc)
    rng = np.random.default_rng(S)
    x = rng.standard_normal(one.n)
    u = okg.seeded_ic(one.n, 3, 0.1)
    for ctx in (one, many):
        ctx.linearize(u)
    # the same rows of the same device factor, gathered: bit-identical V-cycles
    for kind in (_lib.OP_VCYCLE, _lib.OP_SHAT_INV, _lib.OP_SCHUR_TILDE_INV):
        a, b = one.apply(kind, x), many.apply(kind, x)
        assert np.array_equal(a, b), (kind, relerr(b, a))
    u0 = okg.seeded_ic(one.n, 2, 0.0)
    sts = [okg.newton_solve(okg.State(u0, np.zeros(one.n)), okg.build_mesh(dim, n, False), c) for c in (one, many)]
    assert sts[0][1].gmres_iters == sts[1][1].gmres_iters
    assert relerr(sts[1][0].u, sts[0][0].u) <= 1e-10
    many.close()
    one.close()


@pytest.mark.parametrize("dim,n,mcs", [(2, 90, 2116), (3, 30, 4096)])
def test_symmetric_blocks_match_full_rows(dim, n, mcs):
    # one slab: the inverse is stored as its lower block triangle (half the bytes) and
    # both block products are formed from one read; the sums run in another order than
    # the full-row kernel's, so the two agree to rounding
    cfg = cfg_for(dim, n, mcs)
    sym = okg.SchurContext(cfg)
    full = okg.SchurContext(cfg, coarse_split=-1)
    rng = np.random.default_rng(9)
    for _ in range(3):
        xc = rng.uniform(-1, 1, sym.level_sizes[-1])
        a, b = sym.apply(_lib.OP_COARSE_SOLVE, xc), full.apply(_lib.OP_COARSE_SOLVE, xc)
        assert relerr(a, b) <= 1e-14
        assert np.array_equal(a, sym.apply(_lib.OP_COARSE_SOLVE, xc))  # deterministic
    x = rng.uniform(-1, 1, sym.n)
    assert relerr(sym.apply(_lib.OP_VCYCLE, x), full.apply(_lib.OP_VCYCLE, x)) <= 1e-13
    sym.close()
    full.close()
