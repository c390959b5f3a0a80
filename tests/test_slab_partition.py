"""Host logic of the slab decomposition, no GPU needed.

okg_slab_partition is the function every context (thread-per-slab or
process-per-GPU) uses to split the levels into x-plane slabs.  Checked here:
against a restatement of the rule, for tiling / even boundaries / nesting of
coarse ranges / replicated levels, and -- across a world_size-2 gloo process
group, the way bench.py's ranks see it -- that every rank derives the same
hierarchy and that the ranks' slabs tile each split level.
"""
import os
import socket

import pytest

import paper_1603_04570_b200 as okg

CASES = [(2, 64, 2), (2, 64, 3), (2, 128, 4), (2, 2048, 8), (2, 2944, 2), (2, 5888, 8), (3, 16, 2), (3, 32, 4),
         (3, 128, 2), (3, 128, 8), (3, 160, 2), (3, 192, 4), (3, 256, 8)]


REP_MAX = 3_000_000  # okg_params.rep_max_vertices default


def restated(dim, n, S, rank, mcs=500, rep_max=REP_MAX):
    """The partition rule in plain Python."""
    sizes, ln = [], n
    while True:
        sizes.append(ln)
        if not ((ln + 1) ** dim > mcs and ln % 2 == 0):
            break
        ln //= 2
    nlev = len(sizes)
    s0 = n + 1

    def fine(r):
        a = 2 * ((r * s0) // (2 * S))
        b = s0 if r == S - 1 else 2 * (((r + 1) * s0) // (2 * S))
        return a, b

    ranges = [fine(r) for r in range(S)]
    rep, out = nlev, []
    for l in range(nlev):
        small = l > 0 and rep_max > 0 and (sizes[l] + 1) ** dim <= rep_max
        if small or min(b - a for a, b in ranges) < 2 or l + 1 == nlev:
            rep = l
            break
        out.append(ranges[rank])
        ranges = [((a + 1) // 2, (b + 1) // 2) for a, b in ranges]
    out += [(0, sizes[l] + 1) for l in range(rep, nlev)]
    return nlev, rep, out


@pytest.mark.parametrize("rep_max", [0, -1, 40000])
@pytest.mark.parametrize("dim,n,S", CASES)
def test_partition_matches_rule(dim, n, S, rep_max):
    for r in range(S):
        assert okg.slab_partition(dim, n, S, r, rep_max_vertices=rep_max) == \
            restated(dim, n, S, r, rep_max=REP_MAX if rep_max == 0 else rep_max)


def test_replication_threshold_on_baseline_meshes():
    """The cost-model rule on the BASELINE meshes: configs[3] (128^3 on 8 slabs) keeps only the
    finest level split; configs[4] (800^3 on 8) splits 801^3, 401^3, 201^3 and replicates from
    101^3 (1.03 M vertices) down; the old rule (rep_max < 0) splits down to 2 planes per slab."""
    assert okg.slab_partition(3, 128, 8, 0)[1] == 1
    assert okg.slab_partition(3, 128, 8, 0, rep_max_vertices=-1)[1] == 4
    assert okg.slab_partition(3, 800, 8, 3, min_coarse_size=17576)[1] == 3
    assert okg.slab_partition(3, 800, 8, 3, min_coarse_size=17576, rep_max_vertices=-1)[1] == 5
    assert okg.slab_partition(2, 2048, 8, 0)[1] == 1  # 1025^2 = 1.05 M vertices: replicated


@pytest.mark.parametrize("rep_max", [0, -1])
@pytest.mark.parametrize("dim,n,S", CASES)
def test_partition_tiles_and_nests(dim, n, S, rep_max):
    parts = [okg.slab_partition(dim, n, S, r, rep_max_vertices=rep_max) for r in range(S)]
    nlev, rep = parts[0][0], parts[0][1]
    assert 1 <= rep <= nlev - 1
    for l in range(nlev):
        s_l = (n >> l) + 1
        rngs = [p[2][l] for p in parts]
        if l >= rep:
            assert all(rg == (0, s_l) for rg in rngs)
            continue
        assert rngs[0][0] == 0 and rngs[-1][1] == s_l
        for (a, b), (c, d) in zip(rngs, rngs[1:]):
            assert b == c
        assert all(b - a >= 2 for a, b in rngs)
        if l == 0:
            assert all(a % 2 == 0 for a, _ in rngs)
        if l + 1 < rep:  # coarse plane G owned iff fine plane 2G owned
            for (a, b), (ca, cb) in zip(rngs, [p[2][l + 1] for p in parts]):
                assert [g for g in range((n >> (l + 1)) + 1) if a <= 2 * g < b] == list(range(ca, cb))


def test_partition_rejects_too_many_slabs():
    with pytest.raises(okg.InvalidArgument):
        okg.slab_partition(2, 16, 12, 0)
    with pytest.raises(okg.InvalidArgument):
        okg.slab_partition(2, 16, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = {f"{d}-{n}": okg.slab_partition(d, n, world, rank) for d, n, S in CASES}
        everyone = [None] * world
        dist.all_gather_object(everyone, mine)
        ok = True
        for key in mine:
            nlev, rep, _ = everyone[0][key]
            ok &= all(e[key][0] == nlev and e[key][1] == rep for e in everyone)
            for l in range(rep):
                rngs = [e[key][2][l] for e in everyone]
                ok &= all(b == c for (a, b), (c, d) in zip(rngs, rngs[1:]))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_partition_consistent_across_gloo_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
