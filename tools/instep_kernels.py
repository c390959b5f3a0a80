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
    # EXPOSED time: under programmatic dependent launch a kernel's record starts while its predecessor is
    # still running (it sits in griddepcontrol.wait), so durations overlap and their sum exceeds the step.
    # Attribute to each kernel the time from its predecessor's end (or its own start, if later) to its end.
    evs = sorted((ev for ev in prof.events() if ev.device_type.name == "CUDA"), key=lambda e: e.time_range.end)
    prev_end, prev_name, gaps = None, None, {}
    for ev in evs:
        st, en = ev.time_range.start, ev.time_range.end
        ex = en - (st if prev_end is None else max(st, prev_end))
        if prev_end is not None and st > prev_end:  # device idle between two kernels
            gd = gaps.setdefault((prev_name, ev.name), {"n": 0, "us": 0.0})
            gd["n"] += 1
            gd["us"] += st - prev_end
        prev_end, prev_name = en, ev.name
        d = agg[ev.name]
        d["exposed_us"] = d.get("exposed_us", 0.0) + max(0.0, ex)
    instep.gaps = dict(sorted(gaps.items(), key=lambda kv: -kv[1]["us"]))
    return dict(sorted(agg.items(), key=lambda kv: -kv[1].get("exposed_us", kv[1]["total_us"])))


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
    ext = sum(d.get("exposed_us", 0.0) for d in agg.values())
    print(f"# exposed (end-to-end) total {ext / 1e3:.2f} ms; columns: exposed us, share, launches, exposed avg, duration avg")
    for k, d in list(agg.items())[:top]:
        ex = d.get("exposed_us", 0.0)
        print(f"{ex:10.1f} us {100 * ex / max(ext, 1e-9):5.1f}% n={d['n']:6d} exp={ex / max(1, d['n']):7.2f}us "
              f"dur={d['avg_us']:7.2f}us  {k[:80]}")
    gaps = getattr(instep, "gaps", {})
    short = lambda k: k.replace("void ", "").replace("okg::", "").split("(")[0]  # noqa: E731
    # (under CUPTI the gap after a read-back + graph launch is ~250 us; without the profiler it is not on the
    # critical path -- launching the head of the next iteration's graph before the host waits changed nothing)
    print(f"# device idle between kernels: {sum(g['us'] for g in gaps.values()) / 1e3:.2f} ms in "
          f"{sum(g['n'] for g in gaps.values())} gaps; the largest by total (after -> before):")
    for (a, b), gd in list(gaps.items())[:12]:
        print(f"{gd['us']:10.1f} us n={gd['n']:5d} avg={gd['us'] / gd['n']:7.2f}us  {short(a)} -> {short(b)}")
    ctx.close()


if __name__ == "__main__":
    main()
