#!/usr/bin/env python
"""Benchmark: Newton-linear-solve DoFs/s (fp64) of the B200 path.

Default workload = BASELINE.json configs[3] ("C4"): 3D unit cube, 128^3 cubes x
6 Kuhn tetrahedra, P1 (129^3 = 2,146,689 vertices, 4.29 M DoFs), eps=0.02,
sigma=100, m=0, theta=0.5, dt=eps^2, seeded u0 = m + 0.01 U(-1,1) (seed 2,
SURVEY.md 8(d)), w0=0, GMRES(30) rtol 1e-10, newton_tol 1e-8.

A "step" is one implicit timestep = one newton_solve (model.hpp:165-215):
residual, M_E linearisation, block-preconditioned GMRES, update.  W warm-up
timesteps run from the IC, then the state is reset to the IC and K timesteps
are timed (the config's first K timesteps) with CUDA events on the solver's
stream, bracketed by barrier + synchronize.  value = sum(2N * newton_iters) /
time.  The per-step working set (31 Krylov vectors of 2N doubles = 1.1 GB)
is far larger than the 126 MB L2, so no explicit flush is needed.

--impl reference times the reference's own CPU newton_solve (oracle/_ref, the
unmodified okflow headers compiled by oracle/Makefile) on a bounded sample.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Newton-linear-solve DoFs/sec (fp64) at 1/2/4/8 B200; % HBM roofline"

WORKLOADS = {
    # name: (dim, n, eps, m, seed, cpu sample n, description)
    "c4_3d128": (3, 128, 0.02, 0.0, 2, 32,
                 "BASELINE configs[3]: 3D unit cube 128^3 x 6 tets, P1 (2,146,689 vertices, 4,293,378 DoFs), "
                 "eps=0.02 sigma=100 m=0 theta=0.5 dt=eps^2, seed 2, w0=0, GMRES(30) rtol 1e-10, newton_tol 1e-8"),
    "c2_2d2048": (2, 2048, 0.02, 0.0, 0, 128,
                  "BASELINE configs[1] largest: 2D 2048^2 x 2 triangles, P1 (4,198,401 vertices, 8,396,802 DoFs), "
                  "eps=0.02 sigma=100 m=0 theta=0.5 dt=eps^2, seed 0, GMRES(30) rtol 1e-10, newton_tol 1e-8"),
    "c1_2d64": (2, 64, 0.02, 0.0, 0, 64,
                "BASELINE configs[0]: 2D 64^2, seed 0"),
    # configs[4]: 800^3 on 8 GPUs; one GPU runs the per-GPU share, 400^3 (64.5M vertices,
    # 129M DoFs ~ 801^3 / 8), which coarsens to the same 26^3 = 17,576-unknown coarsest level
    # as 800^3 (min_coarse_size raised to admit it, see MIN_COARSE)
    "c5_3d800": (3, 800, 0.02, 0.0, 2, 32,
                 "BASELINE configs[4]: 3D unit cube, 6 tets per cube, P1, eps=0.02 sigma=100 m=0 theta=0.5 "
                 "dt=eps^2, seed 2, w0=0, GMRES(30) rtol 1e-10, newton_tol 1e-8, matrix-free; 800^3 "
                 "(1.03B DoFs) on 8 GPUs, weak slices of ~64.5M vertices per GPU (1 GPU: 400^3, 129M DoFs); "
                 "coarsest 26^3 = 17,576 (min_coarse_size 17576), dense inverse factorised on the device"),
}

# min_coarse_size per workload (default 500 = SolverConfig's): configs[4] needs the
# reference's knob raised so its direct coarse solve admits 26^3 (multigrid.hpp:67-71)
MIN_COARSE = {"c5_3d800": 17576}

# N > 1 (torchrun, one process per GPU, one x-plane slab each): weak scaling keeps
# the vertices per GPU about fixed with meshes whose hierarchy still coarsens to a
# small direct-solve grid (n = 2^k * odd, coarsest <= 2000 vertices)
WEAK_N = {
    "c4_3d128": {1: 128, 2: 160, 4: 192, 8: 256},      # 2.15M, 2.09M, 1.80M, 2.12M vertices per GPU
    "c2_2d2048": {1: 2048, 2: 2944, 4: 4096, 8: 5888},  # 4.20M, 4.34M, 4.20M, 4.33M vertices per GPU
    "c1_2d64": {1: 64, 2: 96, 4: 128, 8: 192},
    "c5_3d800": {1: 400, 2: 512, 4: 640, 8: 800},      # 64.5M, 67.4M, 65.8M, 64.2M vertices per GPU
}

# dominant kernel for the roofline object (top kernel by share of the step in
# the committed ncu launch list, profiles/)
DOMINANT = "resid"  # k_tiled<DIM, L_PLAIN, T_RESID, 8>: 12.6 % (3D 128^3) / 16.5 % (400^3) of a step


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference(dim, n, eps, m, seed, steps, warmup, budget_s=None):
    """The reference's own newton_solve (oracle/_ref) on one host core."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    kind = "ref" if po.available("ref") else "port"
    p = po.baseline_params(dim, n, eps=eps, m=m, kind=kind)
    o = po.Oracle(p, kind)
    u0 = po.seeded_ic(o.n, seed, m, kind)
    w0 = np.zeros(o.n)
    u, w = u0, w0
    for _ in range(warmup):
        u, w, _ = o.newton_solve(u, w)
    u, w = u0, w0
    secs, dofs, iters = 0.0, 0, []
    t_start = time.time()
    for k in range(steps):
        u, w, st = o.newton_solve(u, w)
        secs += st.seconds
        dofs += 2 * o.n * st.newton_iters
        iters.append(st.gmres_iters)
        if budget_s is not None and k >= 1 and time.time() - t_start > budget_s:
            break
    return {"value": dofs / secs, "seconds": secs, "steps": len(iters), "gmres_iters": iters,
            "kind": "reference" if kind == "ref" else "port", "N": o.n,
            "cpu": _cpu_model(), "nproc": os.cpu_count()}


def _ref_worker(args):
    dim, n, eps, m, seed, steps, warmup, budget_s = args
    return cpu_reference(dim, n, eps, m, seed, steps, warmup, budget_s)


def cpu_reference_all_cores(dim, n, eps, m, seed, steps, warmup, budget_s=None, procs=None):
    """The reference's newton_solve on every host core: it is single-threaded
    (proj/README.md:182-184), so the box's CPU throughput is `procs` independent
    solver instances running concurrently (one process each, same sample); the
    aggregate DoF/s is the sum of the instances' rates, each timed by the
    reference's own stats.seconds while all run."""
    import multiprocessing as mp
    procs = procs or os.cpu_count() or 1
    with mp.get_context("spawn").Pool(procs) as pool:
        rs = pool.map(_ref_worker, [(dim, n, eps, m, seed, steps, warmup, budget_s)] * procs)
    r = dict(rs[0])
    r["value"] = sum(x["value"] for x in rs)
    r["per_core"] = [x["value"] for x in rs]
    r["procs"] = procs
    r["steps"] = min(x["steps"] for x in rs)
    r["seconds"] = max(x["seconds"] for x in rs)
    return r


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    dim, n, eps, m, seed, n_cpu, desc = WORKLOADS[args.workload]
    r = cpu_reference_all_cores(dim, n_cpu, eps, m, seed, args.steps, args.warmup)
    sample = (f"{dim}D {n_cpu}^{dim} (same parameters, {r['N']} vertices), {r['steps']} timesteps of the "
              f"reference newton_solve after {args.warmup} warm-up steps, in {r['procs']} concurrent "
              f"single-threaded instances (the reference has no threading, proj/README.md:182-184; one "
              f"instance per host core, aggregate = sum of their rates; per instance "
              f"{min(r['per_core']):.3g}-{max(r['per_core']):.3g} DoF/s); CPU {r['cpu']}, nproc {r['nproc']}")
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "DoF/s", "n_gpus": world,
        "steps": r["steps"], "warmup": args.warmup, "ms_per_step": 1e3 * r["seconds"] / r["steps"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded IC, SURVEY.md 8(d))",
        "config": {"workload": args.workload, "description": desc, "sample_n": n_cpu},
        "cpu_baseline": {"value": r["value"], "unit": "DoF/s", "cores": r["procs"], "kind": r["kind"],
                         "sample": sample},
        "e2e": {"value": r["value"], "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gmres_iters": r["gmres_iters"],
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="okg", choices=["okg", "reference"])
    ap.add_argument("--workload", default="c4_3d128", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of reference CPU work (cpu_baseline)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = mesh grows with N (WEAK_N), strong = the workload's mesh split N ways")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    device = local_rank if world > 1 else 0

    import paper_1603_04570_b200 as okg
    from paper_1603_04570_b200 import _lib
    import ctypes as C

    dim, n, eps, m, seed, n_cpu, desc = WORKLOADS[args.workload]
    if (world > 1 and args.scaling == "weak") or (world == 1 and args.workload == "c5_3d800"):
        n = WEAK_N[args.workload].get(world)
        if n is None:
            raise SystemExit(f"--scaling weak: no mesh for {world} GPUs (have {sorted(WEAK_N[args.workload])})")
    cfg = okg.SolverConfig(dim=dim, n=n, eps=eps, m=m, sigma=100.0, theta=0.5, dt=eps * eps,
                           newton_tol=1e-8, gmres_tol=1e-10, gmres_restart=30,
                           min_coarse_size=MIN_COARSE.get(args.workload, 500))
    t0 = time.time()
    if world > 1:
        # one slab per process: rank 0 makes the NCCL id of the solver's own communicator
        idt = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{device}")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(okg.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        ctx = okg.SchurContext(cfg, device=device, rank=rank, nranks=world, nccl_id=bytes(idt.cpu().numpy()))
    else:
        ctx = okg.SchurContext(cfg, device=device)
    setup_s = time.time() - t0
    N = ctx.n
    u0 = okg.seeded_ic(N, seed, m)
    w0 = np.zeros(N)
    ic = okg.State(u0, w0)

    sp = C.c_void_p()
    _lib.check(_lib.lib.okg_stream(ctx.handle, C.byref(sp)))
    stream = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", device))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(device)

    # ---- warm-up ----
    ctx.set_state(ic)
    for _ in range(args.warmup):
        ctx.step_resident()

    # ---- timed: device-resident inputs ----
    ctx.set_state(ic)
    clocks = ClockSampler(device)
    barrier()
    clocks.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    stats = [ctx.step_resident() for _ in range(args.steps)]
    ev1.record(stream)
    barrier()
    clocks_info = clocks.stop()
    t_ms = ev0.elapsed_time(ev1)
    dofs = sum(2 * N * s.newton_iters for s in stats)
    launches = sum(s.kernel_launches for s in stats)
    t_tensor = torch.tensor([t_ms], dtype=torch.float64, device=f"cuda:{device}")
    if dist is not None:
        dist.all_reduce(t_tensor, op=dist.ReduceOp.MAX)
    t_max_ms = float(t_tensor.item())
    value = dofs / (t_max_ms * 1e-3)  # dofs counts the whole mesh (all slabs) once

    # ---- e2e: through the C ABI with pinned host buffers, H2D/D2H inside ----
    hu_in = torch.from_numpy(u0.copy()).pin_memory()
    hw_in = torch.from_numpy(w0.copy()).pin_memory()
    hu_out = torch.empty(N, dtype=torch.float64).pin_memory()
    hw_out = torch.empty(N, dtype=torch.float64).pin_memory()
    dp = lambda t: C.cast(C.c_void_p(t.data_ptr()), _lib._dp)  # noqa: E731
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_dofs = 0
    for _ in range(args.steps):
        ss = _lib.StepStats()
        _lib.check(_lib.lib.okg_newton_step_host(ctx.handle, dp(hu_in), dp(hw_in), dp(hu_out), dp(hw_out),
                                                 C.byref(ss)))
        e2e_dofs += 2 * N * ss.newton_iters
        hu_in, hu_out = hu_out, hu_in
        hw_in, hw_out = hw_out, hw_in
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    e2e_t = torch.tensor([e2e_ms], dtype=torch.float64, device=f"cuda:{device}")
    if dist is not None:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = e2e_dofs / (float(e2e_t.item()) * 1e-3)
    lt = torch.tensor([launches], dtype=torch.int64, device=f"cuda:{device}")
    if dist is not None:
        dist.all_reduce(lt)  # kernels of every rank
    launches = int(lt.item())

    # ---- per-kernel live timing (CUDA events on the solver stream) ----
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        try:
            peak = float(json.load(open(peaks_path))["hbm_gbs"])
            peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)"
        except Exception:
            pass
    kernels = {}
    ctx.linearize(u0)
    for kid, name in enumerate(_lib.KT_NAMES):
        ms, by = C.c_double(), C.c_double()
        st = _lib.lib.okg_kernel_timing(ctx.handle, kid, 50, C.byref(ms), C.byref(by))
        if st == 0:
            kernels[name] = {"avg_us": ms.value * 1e3, "alg_bytes": by.value,
                             "gbs": by.value / (ms.value * 1e-3) / 1e9}
    ctx.clear_linearization()
    dom = kernels.get(DOMINANT)
    roofline = None
    if dom:
        roofline = {"bound": "hbm", "kernel": f"{DOMINANT} (fine-level residual sweep b - Shat_0 x, k_tiled<{dim}, L_PLAIN, T_RESID, 8>)",
                    "achieved": dom["gbs"], "peak": peak, "unit": "GB/s", "frac": dom["gbs"] / peak,
                    "peak_source": peak_src, "traffic": None,
                    "alg_bytes_per_launch": dom["alg_bytes"], "avg_launch_us": dom["avg_us"]}
        prof = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(prof):
            try:
                tr = json.load(open(prof)).get(args.workload, {}).get(DOMINANT)
                if tr:
                    roofline["traffic"] = tr
            except Exception:
                pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference_all_cores(dim, n_cpu, eps, m, seed, 100, 0, budget_s=args.cpu_budget)
            cpu = {"value": r["value"], "unit": "DoF/s", "cores": r["procs"], "kind": r["kind"],
                   "sample": (f"{dim}D {n_cpu}^{dim} ({r['N']} vertices), >= {r['steps']} timesteps of the "
                              f"reference newton_solve from the same seeded IC in each of {r['procs']} concurrent "
                              f"single-threaded instances (one per host core; the reference has no threading), "
                              f"each timed by its own stats.seconds, aggregate = sum of rates; CPU {r['cpu']}, "
                              f"nproc {r['nproc']}")}
        except Exception as e:  # report, never fail the GPU line
            cpu = {"value": None, "unit": "DoF/s", "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded IC u0 = m + 0.01 U(-1,1), SURVEY.md 8(d); no dataset involved)",
            "config": {"workload": args.workload, "description": desc, "dim": dim, "n": n, "dofs": 2 * N,
                       "parallelism": "1 GPU" if world == 1 else
                       (f"{world} x-plane slabs, one per GPU/process; ghost planes by NCCL send/recv, "
                        f"Krylov sums by NCCL allreduce; planes per rank {ctx.slab_planes}"),
                       "l2": f"per-step working set ({31 * 2 * N * 8 / 1e9:.1f} GB Krylov basis) >> 126 MB L2; no flush",
                       "setup_s": setup_s, "levels": ctx.level_sizes},
            "newton_iters": [s.newton_iters for s in stats],
            "gmres_iters": [s.gmres_iters for s in stats],
            "clocks": clocks_info,
            "e2e": {"value": e2e_value, "unit": "DoF/s", "h2d_bytes_per_step": 2 * N * 8,
                    "d2h_bytes_per_step": 2 * N * 8},
            "gpu_launches": launches,
            "roofline": roofline,
            "kernels": kernels,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
