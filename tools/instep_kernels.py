"""In-step per-kernel device times of one Newton timestep (CUPTI activity records
via torch.profiler/kineto), for the roofline cross-check of bench.py.

usage: python tools/instep_kernels.py DIM N [steps] [top]
Prints one JSON object: {kernel name: {"n": launches, "avg_us": .., "total_us": ..}}
plus the step total, sorted by total time.  Run it alone (never inside a timed region).
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def instep(ctx, steps=1):
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            ctx.step_resident()
        torch.cuda.synchronize()
    agg = {}
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        name = ev.name
        d = agg.setdefault(name, {"n": 0, "total_us": 0.0})
        d["n"] += 1
        d["total_us"] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    for d in agg.values():
        d["avg_us"] = d["total_us"] / max(1, d["n"])
    return dict(sorted(agg.items(), key=lambda kv: -kv[1]["total_us"]))


def main():
    import paper_1603_04570_b200 as okg
    dim, n = int(sys.argv[1]), int(sys.argv[2])
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    cfg = okg.SolverConfig(dim=dim, n=n, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30,
                           min_coarse_size=int(os.environ.get("OKG_MIN_COARSE", "500")))
    ctx = okg.SchurContext(cfg)
    ic = okg.State(okg.seeded_ic(ctx.n, 2 if dim == 3 else 0, 0.0), np.zeros(ctx.n))
    ctx.set_state(ic)
    for _ in range(2):
        ctx.step_resident()
    ctx.set_state(ic)
    agg = instep(ctx, steps)
    tot = sum(d["total_us"] for d in agg.values())
    print(f"# total {tot / 1e3:.2f} ms over {sum(d['n'] for d in agg.values())} kernels, {steps} step(s)")
    for k, d in list(agg.items())[:top]:
        print(f"{d['total_us']:10.1f} us {100 * d['total_us'] / tot:5.1f}% n={d['n']:6d} avg={d['avg_us']:8.2f}us  {k[:90]}")
    ctx.close()


if __name__ == "__main__":
    main()
