"""The multi-slab DATA PLANE protocol over a real world_size-2 gloo group, on the CPU.

The CUDA slab path (csrc/okg_host.cu: mg_level, exchange, allgather_planes, allreduce)
cannot run here, but what makes it correct is a protocol: which planes a slab owns on
every level (okg_slab_partition, the product's own function), that ONE ghost plane per
side is enough for the stencil, for P^T (after the residual's exchange) and for P (after
the coarse correction's exchange), where the exchanges sit in the V(2,2) cycle, the
restriction into the first replicated level followed by an all-gather of plane ranges,
and rank-ordered reductions.  This test restates that protocol in numpy on top of the
oracle's own level operators (dense S_l and P_l from oracle/okport.c), runs it with two
gloo ranks that really exchange planes through torch.distributed, and checks that

* no value a slab was never sent is ever used: everything outside a slab's owned + ghost
  planes is NaN, and every operator row is checked to touch local planes only;
* the two-slab V-cycle equals the one-domain V-cycle of the same numpy code (<= 1e-13)
  and the oracle's v_cycle (multigrid.hpp:97-129, <= 1e-10);
* the rank-ordered all-reduced dot products equal the one-domain dot products.

Both partition depths run: split as deep as two planes per slab, and the default
replication rule (every level below the finest replicated at these sizes).
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_1603_04570_b200 as okg  # noqa: E402

CASES = [(2, 16, 20, -1), (2, 32, 30, -1), (3, 8, 20, -1), (2, 16, 20, 0), (3, 8, 20, 0)]
OMEGA = 2.0 / 3.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class Hier:
    """Dense level operators of the oracle (the port), identical on every rank."""

    def __init__(self, dim, n, mcs):
        import pyoracle as po
        self.po = po
        self.o = po.Oracle(po.baseline_params(dim, n, kind="port", min_coarse_size=mcs, mg_omega=OMEGA), "port")
        self.dim, self.L = dim, self.o.levels
        self.N = [self.o.level_size(l) for l in range(self.L)]
        self.s = [int(round(N ** (1.0 / dim))) for N in self.N]
        self.A = [self.o.level_dense(l) for l in range(self.L)]
        self.P = []
        for l in range(self.L - 1):
            P = np.empty((self.N[l], self.N[l + 1]))
            for j in range(self.N[l + 1]):
                e = np.zeros(self.N[l + 1])
                e[j] = 1.0
                P[:, j] = self.o.apply(po.PROLONG, e, level=l)
            self.P.append(P)

    def ps(self, l):
        return self.s[l] ** (self.dim - 1)

    def planes(self, l, a, b):
        """vertex indices of x-planes [a, b) of level l (x is the slowest index)."""
        a, b = max(a, 0), min(b, self.s[l])
        return np.arange(a * self.ps(l), b * self.ps(l))

    # ---- one-domain V(2,2) cycle in this file's arithmetic
    def vcycle(self, l, b):
        A = self.A[l]
        if l == self.L - 1:
            return np.linalg.solve(A, b)
        wd = OMEGA / np.diag(A)
        e = wd * b
        e = e + wd * (b - A @ e)
        bc = self.P[l].T @ (b - A @ e)
        e = e + self.P[l] @ self.vcycle(l + 1, bc)
        for _ in range(2):
            e = e + wd * (b - A @ e)
        return e


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    report = []
    try:
        for dim, n, mcs, rep_max in CASES:
            H = Hier(dim, n, mcs)
            nlev, rep, rng = okg.slab_partition(dim, n, world, rank, min_coarse_size=mcs, rep_max_vertices=rep_max)
            allr = [okg.slab_partition(dim, n, world, r, min_coarse_size=mcs, rep_max_vertices=rep_max)[2]
                    for r in range(world)]
            assert nlev == H.L

            def own(l):
                return H.planes(l, *rng[l])

            def loc(l):  # owned + one ghost plane per side
                return H.planes(l, rng[l][0] - 1, rng[l][1] + 1)

            def exchange(l, v):
                """boundary planes out, ghost planes in (okg_host.cu exchange())."""
                lo, hi = rng[l]
                reqs, bufs = [], []
                for nb, send_pl, recv_pl in ((rank - 1, lo, lo - 1), (rank + 1, hi - 1, hi)):
                    if nb < 0 or nb >= world:
                        continue
                    out = torch.from_numpy(v[H.planes(l, send_pl, send_pl + 1)].copy())
                    buf = torch.empty(H.ps(l), dtype=torch.float64)
                    reqs += [dist.isend(out, nb), dist.irecv(buf, nb)]
                    bufs.append((recv_pl, buf))
                for r in reqs:
                    r.wait()
                for pl, buf in bufs:
                    v[H.planes(l, pl, pl + 1)] = buf.numpy()

            def rows(M, r, c, x):
                """(M x)[r] from x[c] only; the rest of every row must be structurally zero."""
                mask = np.ones(M.shape[1], bool)
                mask[c] = False
                assert not np.any(M[np.ix_(r, np.nonzero(mask)[0])]), "operator row reaches past the ghost planes"
                return M[np.ix_(r, c)] @ x[c]

            def vc_dist(l, b):
                """mg_level of okg_host.cu on this slab: b valid on owned planes, NaN elsewhere."""
                if l >= rep:
                    return H.vcycle(l, b)  # replicated: every slab runs the whole level
                A, o_, c_ = H.A[l], own(l), loc(l)
                wd = OMEGA / np.diag(A)
                nanv = lambda: np.full(H.N[l], np.nan)  # noqa: E731
                exchange(l, b)
                e1 = nanv()
                e1[c_] = wd[c_] * b[c_]                       # staged on the halo too (L_JAC0)
                cur = nanv()
                cur[o_] = e1[o_] + wd[o_] * (b[o_] - rows(A, o_, c_, e1))
                exchange(l, cur)
                res = nanv()
                res[o_] = b[o_] - rows(A, o_, c_, cur)
                exchange(l, res)
                # coarse vertices G with fine plane 2G owned
                clo, chi = (rng[l][0] + 1) // 2, (rng[l][1] + 1) // 2
                cown = H.planes(l + 1, clo, chi)
                bc = np.full(H.N[l + 1], np.nan)
                bc[cown] = rows(H.P[l].T, cown, c_, res)
                if l + 1 >= rep:  # first replicated level: all-gather the slabs' plane ranges
                    parts = [None] * world
                    dist.all_gather_object(parts, (clo, chi, bc[cown]))
                    for a, b2, vals in parts:
                        bc[H.planes(l + 1, a, b2)] = vals
                    assert not np.isnan(bc).any()
                else:
                    assert (clo, chi) == tuple(rng[l + 1])
                ec = vc_dist(l + 1, bc)
                if l + 1 < rep:
                    exchange(l + 1, ec)
                    cl = loc(l + 1)
                else:
                    cl = np.arange(H.N[l + 1])
                exchange(l, cur)
                s_ = nanv()
                s_[c_] = cur[c_] + rows(H.P[l], c_, cl, ec)   # e + P e_c staged on the halo (L_PROLONG)
                y = nanv()
                y[o_] = s_[o_] + wd[o_] * (b[o_] - rows(A, o_, c_, s_))
                exchange(l, y)
                out = nanv()
                out[o_] = y[o_] + wd[o_] * (b[o_] - rows(A, o_, c_, y))
                return out

            gen = np.random.default_rng(100 * dim + n)
            b = gen.uniform(-1, 1, H.N[0])
            z = gen.uniform(-1, 1, H.N[0])
            ref = H.vcycle(0, b)
            bl = np.full(H.N[0], np.nan)
            bl[own(0)] = b[own(0)]
            mine = vc_dist(0, bl)
            assert not np.isnan(mine[own(0)]).any(), "a value that was never exchanged reached an owned vertex"
            err = np.linalg.norm(mine[own(0)] - ref[own(0)]) / np.linalg.norm(ref)
            # rank-ordered reduction of the partial dot products (allreduce of okg_host.cu)
            part = torch.tensor([float(np.dot(b[own(0)], z[own(0)]))], dtype=torch.float64)
            parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, part)
            dot = sum(float(p[0]) for p in parts)  # rank order: the same bits on every rank
            derr = abs(dot - float(np.dot(b, z))) / abs(float(np.dot(b, z)))
            oerr = np.linalg.norm(ref - H.o.apply(H.po.VCYCLE, b)) / np.linalg.norm(ref)
            tiles = all(allr[r][0][1] == allr[r + 1][0][0] for r in range(world - 1))
            report.append((dim, n, rep_max, rep, float(err), float(derr), float(oerr), bool(tiles)))
        q.put((rank, report))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, f"{type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


def test_two_slab_vcycle_protocol_over_gloo():
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank in (0, 1):
        assert isinstance(res[rank], list), res[rank]
        assert len(res[rank]) == len(CASES)
        for (dim, n, rep_max, rep, err, derr, oerr, tiles), case in zip(res[rank], CASES):
            assert tiles
            assert err <= 1e-13, (rank, case, err)
            assert derr <= 1e-14, (rank, case, derr)
            assert oerr <= 1e-10, (rank, case, oerr)
            # deep split: at least two split levels; default rule: only the finest is split
            assert rep >= 2 if rep_max < 0 else rep == 1
