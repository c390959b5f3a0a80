"""Slab decomposition against the one-slab solve.

The mesh is split into x-plane slabs, each with its own host thread, CUDA
stream and device buffers (+1 ghost plane per side), exchanging ghost planes
before every stencil kernel and allreducing (in rank order) every partial sum.
Here all slabs share cuda:0 -- ordering is CUDA events + host barriers, no
kernel waits on another -- so this runs the exact multi-slab code path of the
multi-GPU configuration on one GPU.

What must hold ("iteration counts must match 1-GPU exactly,
+-rounding"):
* every pointwise/stencil operator and the whole multigrid V-cycle agree
  BIT-EXACTLY with the one-slab context (same per-vertex arithmetic; the
  replicated coarse levels are gathered, not recomputed);
* operators that depend on the Lanczos bounds (Chebyshev) agree to rounding
  (the bounds' dot products are summed in another order);
* GMRES and Newton take the same number of iterations and agree to 1e-10.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import relerr

import paper_1603_04570_b200 as okg
from paper_1603_04570_b200 import _lib

pytestmark = pytest.mark.gpu

EXACT = [("M", _lib.OP_M), ("K", _lib.OP_K), ("A", _lib.OP_A), ("SHAT0", _lib.OP_SHAT),
         ("VCYCLE", _lib.OP_VCYCLE), ("SHAT_INV", _lib.OP_SHAT_INV), ("ME", _lib.OP_ME), ("C", _lib.OP_C),
         ("SCHUR_TILDE_INV", _lib.OP_SCHUR_TILDE_INV), ("NONLINEAR", _lib.OP_NONLINEAR)]
ROUNDING = [("CHEB_M", _lib.OP_CHEB_M), ("CHEB_A", _lib.OP_CHEB_A), ("SCHUR", _lib.OP_SCHUR),
            ("S_INV_APPROX", _lib.OP_S_INV_APPROX)]

MODES = {"default": {}, "tiled": dict(tiled_min_n=2, mg_fuse=1), "plain": dict(tiled_min_n=-1, mg_fuse=-1)}

# (dim, n, slabs, rep_max_vertices): -1 splits every level down to 2 planes per slab (the deep
# hierarchy of ghost exchanges), 0 is the default cost-model rule (small levels replicated)
CASES = [(2, 64, 2, -1), (2, 64, 3, -1), (2, 128, 4, -1), (3, 16, 2, -1), (3, 32, 3, -1), (3, 32, 4, -1),
         (2, 128, 4, 0), (3, 32, 4, 0), (3, 32, 2, 2000)]


def cfg_for(dim, n):
    return okg.SolverConfig(dim=dim, n=n, m=0.0, eps=0.02, dt=4e-4, gmres_tol=1e-10, gmres_restart=30,
                            newton_tol=1e-8)


@pytest.fixture(scope="module", params=[(c, m) for c in CASES for m in MODES],
                ids=lambda p: f"{p[0][0]}d{p[0][1]}-s{p[0][2]}-r{p[0][3]}-{p[1]}")
def pair(request):
    (dim, n, S, rep_max), mode = request.param
    cfg = cfg_for(dim, n)
    # the collapsed bottom of the V-cycle needs whole (replicated) levels; a split level
    # would keep the recursive cycle on the slabs -- compare like with like
    one = okg.SchurContext(cfg, mg_collapse=-1, **MODES[mode])
    many = okg.SchurContext(cfg, nslabs=S, mg_collapse=-1, rep_max_vertices=rep_max, **MODES[mode])
    many.rep_max = rep_max
    yield dim, n, S, one, many
    many.close()
    one.close()


def test_partition(pair):
    dim, n, S, one, many = pair
    assert many.nslabs == S and one.nslabs == 1
    planes = many.slab_planes
    assert planes[0][0] == 0 and planes[-1][1] == n + 1
    for (a, b), (c, d) in zip(planes, planes[1:]):
        assert b == c and b % 2 == 0  # contiguous, even boundaries (P / P^T nest)
    assert all(b - a >= 2 for a, b in planes)
    assert 1 <= many.rep_level <= many.levels - 1
    assert many.level_sizes == one.level_sizes
    assert one.rep_level == one.levels


def test_scalars(pair):
    dim, n, S, one, many = pair
    assert many.c == one.c and many.eps_sqrt_c == one.eps_sqrt_c
    assert abs(many.lambda_lo - one.lambda_lo) <= 1e-12 * one.lambda_lo
    assert abs(many.lambda_hi - one.lambda_hi) <= 1e-12 * one.lambda_hi


def test_operators(pair):
    dim, n, S, one, many = pair
    N = one.n
    rng = np.random.default_rng(7)
    x = rng.standard_normal(N)
    x2 = rng.standard_normal(2 * N)
    u = okg.seeded_ic(N, 3, 0.1) + 0.3 * rng.standard_normal(N)
    for ctx in (one, many):
        ctx.linearize(u)
    for key, kind in EXACT:
        arg = u if kind == _lib.OP_NONLINEAR else x
        a, b = one.apply(kind, arg), many.apply(kind, arg)
        assert np.array_equal(a, b), (key, relerr(b, a))
    for key, kind in ROUNDING:
        assert relerr(many.apply(kind, x), one.apply(kind, x)) <= 1e-12, key
    assert np.array_equal(many.apply(_lib.OP_JACOBIAN, x2), one.apply(_lib.OP_JACOBIAN, x2))
    assert relerr(many.apply(_lib.OP_BLOCK, x2), one.apply(_lib.OP_BLOCK, x2)) <= 1e-12
    # residual: pointwise + stencil, bit-exact
    old = okg.State(okg.seeded_ic(N, 5, 0.0), np.zeros(N))
    nxt = okg.State(old.u + 1e-3 * rng.standard_normal(N), rng.standard_normal(N))
    r1a, r2a = one.residual(nxt, old)
    r1b, r2b = many.residual(nxt, old)
    assert np.array_equal(r1a, r1b) and np.array_equal(r2a, r2b)


def test_gmres(pair):
    dim, n, S, one, many = pair
    N = one.n
    rng = np.random.default_rng(11)
    u = okg.seeded_ic(N, 2, 0.0)
    b = rng.standard_normal(2 * N)
    res = []
    for ctx in (one, many):
        ctx.linearize(u)
        res.append(ctx.gmres(b, 1e-10, 200, 30))
    assert res[0].converged and res[1].converged
    assert res[1].iterations == res[0].iterations
    assert relerr(res[1].x, res[0].x) <= 1e-10


def test_newton_steps(pair):
    dim, n, S, one, many = pair
    N = one.n
    st0 = okg.State(okg.seeded_ic(N, 2, 0.0), np.zeros(N))
    out = []
    for ctx in (one, many):
        ctx.set_state(st0)
        stats = [ctx.step_resident() for _ in range(2)]
        out.append((stats, ctx.get_state()))
    (sa, xa), (sb, xb) = out
    for a, b in zip(sa, sb):
        assert a.converged and b.converged
        assert a.newton_iters == b.newton_iters
        assert a.gmres_iters == b.gmres_iters
    assert xb.step == xa.step == 2 and xb.t == xa.t
    assert relerr(xb.u, xa.u) <= 1e-10 and relerr(xb.w, xa.w) <= 1e-10


def test_newton_host_entry(pair):
    dim, n, S, one, many = pair
    N = one.n
    u0 = okg.seeded_ic(N, 9, 0.0)
    w0 = np.zeros(N)
    res = []
    for ctx in (one, many):
        un, wn = np.empty(N), np.empty(N)
        ss = _lib.StepStats()
        okg.check(_lib.lib.okg_newton_step_host(ctx.handle, u0.ctypes.data_as(_lib._dp), w0.ctypes.data_as(_lib._dp),
                                                un.ctypes.data_as(_lib._dp), wn.ctypes.data_as(_lib._dp),
                                                C.byref(ss)))
        res.append((ss.newton_iters, list(ss.gmres_iters[:ss.newton_iters]), un, wn))
    assert res[0][:2] == res[1][:2]
    assert relerr(res[1][2], res[0][2]) <= 1e-10 and relerr(res[1][3], res[0][3]) <= 1e-10


def test_multislab_rejects_device_pointer_api(pair):
    dim, n, S, one, many = pair
    x = okg.DeviceArray(many.n)
    y = okg.DeviceArray(many.n)
    with pytest.raises(okg.InvalidArgument):
        many.apply_dev(_lib.OP_M, x, y)
    with pytest.raises(okg.InvalidArgument):
        many.apply(_lib.OP_PROLONG, np.zeros(many.level_sizes[1]), level=0)


def test_too_many_slabs():
    with pytest.raises(okg.OkgError):
        okg.SchurContext(cfg_for(2, 16), nslabs=12)
    with pytest.raises(okg.InvalidArgument):
        okg.SchurContext(cfg_for(2, 64), nslabs=17)


def test_full_size_3d128_two_slabs():
    """BASELINE config 4 (3D 128^3) split in two: same Newton/GMRES iteration counts."""
    cfg = okg.SolverConfig(dim=3, n=128, m=0.0, eps=0.02, dt=0.02 ** 2, gmres_tol=1e-10, gmres_restart=30)
    N = cfg.num_vertices()
    st0 = okg.State(okg.seeded_ic(N, 2, 0.0), np.zeros(N))
    out = []
    for S in (1, 2):
        ctx = okg.SchurContext(cfg, nslabs=S)
        ctx.set_state(st0)
        s = ctx.step_resident()
        out.append((s.newton_iters, s.gmres_iters, ctx.get_state()))
        ctx.close()
    assert out[0][0] == out[1][0] and out[0][1] == out[1][1]
    assert relerr(out[1][2].u, out[0][2].u) <= 1e-10


def test_rank_context_one_process():
    """okg_create_rank (one process per GPU, NCCL transport) with a single rank: a
    real NCCL communicator is created; results equal the ordinary context."""
    cfg = cfg_for(2, 64)
    one = okg.SchurContext(cfg)
    r0 = okg.SchurContext(cfg, rank=0, nranks=1, nccl_id=okg.nccl_unique_id())
    assert r0.nslabs == 1 and r0.slab_planes == [(0, 65)]
    N = one.n
    st0 = okg.State(okg.seeded_ic(N, 2, 0.0), np.zeros(N))
    out = []
    for ctx in (one, r0):
        ctx.set_state(st0)
        s = ctx.step_resident()
        out.append((s.newton_iters, s.gmres_iters, ctx.get_state()))
    assert out[0][:2] == out[1][:2]
    assert np.array_equal(out[0][2].u, out[1][2].u)
    r0.close()
    one.close()


def test_create_rank_argument_checks():
    cfg = cfg_for(2, 64)
    with pytest.raises(okg.InvalidArgument):
        okg.SchurContext(cfg, rank=2, nranks=2, nccl_id=bytes(128))
    with pytest.raises(okg.InvalidArgument):
        okg.SchurContext(cfg, rank=0, nranks=2, nccl_id=None)
