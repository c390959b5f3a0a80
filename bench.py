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

--gpus N > 1 without WORLD_SIZE in the environment re-launches this script
under torchrun (one process per GPU, 127.0.0.1 rendezvous).  configs[3]
(c4_3d128, the default) is the SAME 128^3 problem on 1/2/4/8 GPUs (strong
scaling, x-plane slabs); configs[4] (c5_3d800) grows the mesh with N (weak).

--impl reference times the reference's own CPU newton_solve (oracle/_ref, the
unmodified okflow headers compiled by oracle/Makefile) on the SAME workload
(setup untimed, then its first timestep timed by the reference's own
stats.seconds): one instance alone (one host core), then as many concurrent
single-threaded instances as host cores and RAM allow (the value: the box's
whole CPU).

Per-kernel numbers (`kernels`, `roofline`): every fine-level kernel is timed
(a) in-step -- CUPTI activity records (torch.profiler) of one extra timestep
after the timed region, the launch with the largest grid of that kernel's
template (the fine level); `roofline.achieved` uses this time -- and (b) alone
and L2-cold with CUDA events (okg_kernel_timing_ex: a 2 x L2 scratch write
before every launch, no PDL).
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

# N > 1 default: configs[3] is the same 128^3 problem on 2/4/8 GPUs (strong);
# configs[4] is weak-scaled (100^3 cells per GPU-equivalent share)
DEFAULT_SCALING = {"c4_3d128": "strong", "c2_2d2048": "strong", "c1_2d64": "strong", "c5_3d800": "weak"}

# (the roofline kernel is chosen live: the fine-level kernel with the largest share
#  of the in-step device time)


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


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _mem_available():
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                return int(ln.split()[1]) * 1024
    except Exception:
        pass
    return 0


# peak RSS of one reference instance per vertex (7.19 GB at 3D 128^3,
# 4.68 GB at 2D 2048^2), rounded up
REF_BYTES_PER_VERTEX = {2: 1200, 3: 3600}


def ref_instance(args):
    """One reference instance (oracle/_ref: the unmodified okflow headers): build_mesh +
    assemble_operators + make_schur_context (untimed), then newton_solve timesteps from
    the seeded IC until `budget_s` of solve time (at least one), each timed by the
    reference's own stats.seconds (model.hpp:168,211-213)."""
    dim, n, eps, m, seed, min_coarse, budget_s, max_steps = args
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    kind = "ref" if po.available("ref") else "port"
    t0 = time.time()
    p = po.baseline_params(dim, n, eps=eps, m=m, kind=kind, min_coarse_size=min_coarse)
    o = po.Oracle(p, kind)
    setup_s = time.time() - t0
    u = po.seeded_ic(o.n, seed, m, kind)
    w = np.zeros(o.n)
    secs, dofs, iters = 0.0, 0, []
    while True:
        u, w, st = o.newton_solve(u, w)
        secs += st.seconds
        dofs += 2 * o.n * st.newton_iters
        iters.append(st.gmres_iters)
        if secs >= budget_s or len(iters) >= max_steps:
            break
    o.close()
    return {"value": dofs / secs, "seconds": secs, "steps": len(iters), "gmres_iters": iters,
            "kind": "reference" if kind == "ref" else "port", "N": int(o.n), "setup_s": setup_s}


def ref_concurrent(dim, n, eps, m, seed, min_coarse, budget_s, max_steps, procs):
    """`procs` single-threaded reference instances at once (one process each): the
    reference has no threading (proj/README.md:182-184), so this is the box's whole
    CPU.  Aggregate = sum of the instances' rates."""
    import multiprocessing as mp
    a = (dim, n, eps, m, seed, min_coarse, budget_s, max_steps)
    with mp.get_context("spawn").Pool(procs) as pool:
        rs = pool.map(ref_instance, [a] * procs)
    return {"value": sum(x["value"] for x in rs), "per_instance": [x["value"] for x in rs], "procs": procs,
            "steps": min(x["steps"] for x in rs), "seconds": max(x["seconds"] for x in rs),
            "gmres_iters": rs[0]["gmres_iters"], "kind": rs[0]["kind"], "N": rs[0]["N"],
            "setup_s": max(x["setup_s"] for x in rs)}


def workload_mesh(workload, world, scaling):
    dim, n, eps, m, seed, n_cpu, desc = WORKLOADS[workload]
    if (world > 1 and scaling == "weak") or (world == 1 and workload == "c5_3d800"):
        n = WEAK_N[workload].get(world)
        if n is None:
            raise SystemExit(f"--scaling weak: no mesh for {world} GPUs (have {sorted(WEAK_N[workload])})")
    return dim, n


def workload_config(workload, dim, n):
    """The workload's config object -- identical in both arms (GPU and --impl reference)."""
    N = (n + 1) ** dim
    return {"workload": workload, "description": WORKLOADS[workload][6], "dim": dim, "n": n, "dofs": 2 * N,
            "l2": f"inputs larger than L2: per-step working set ({31 * 2 * N * 8 / 1e9:.2f} GB Krylov basis "
                  f"+ level vectors) >> 126 MB L2; no flush"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    dim, _, eps, m, seed, _, desc = WORKLOADS[args.workload]
    dim, n = workload_mesh(args.workload, world, args.scaling)
    cfg = workload_config(args.workload, dim, n)
    base = {"impl": "reference", "metric": METRIC, "unit": "DoF/s", "n_gpus": world, "config": cfg}
    if args.workload == "c5_3d800":
        base["unavailable"] = ("the reference cannot run configs[4]: its coarsest 26^3 = 17,576 exceeds the "
                               "dense cap (ConfigError, multigrid.hpp:52,67-71); with the cap raised its host "
                               "Cholesky of 17,576^2 and int32 CSR put it at hours per step")
        print(json.dumps(base), flush=True)
        return 0
    N = (n + 1) ** dim
    need = REF_BYTES_PER_VERTEX[dim] * N + (256 << 20)
    ncpu = os.cpu_count() or 1
    procs = max(1, min(ncpu, int(0.85 * _mem_available() // need) if _mem_available() else 1))
    if args.ref_procs:
        procs = args.ref_procs
    a = (dim, n, eps, m, seed, MIN_COARSE.get(args.workload, 500), args.ref_budget, max(1, args.steps))
    single = None
    if world == 1 and not args.ref_no_single:
        single = ref_instance(a)
    r = ref_concurrent(*a, procs)
    cpu = _cpu_model()
    sample = (f"the workload itself ({dim}D {n}^{dim}, {N} vertices): setup untimed, then the first "
              f"{r['steps']} timestep(s) of the reference newton_solve from the seeded IC, timed by its own "
              f"stats.seconds, in {procs} concurrent single-threaded instances (the reference has no threading, "
              f"proj/README.md:182-184; {procs} = min(nproc {ncpu}, 85% of MemAvailable / "
              f"{need / 1e9:.1f} GB per instance)); aggregate = sum of the instances' rates, per instance "
              f"{min(r['per_instance']):.3g}-{max(r['per_instance']):.3g} DoF/s; CPU {cpu}")
    line = dict(base)
    line.update({
        "value": r["value"], "steps": r["steps"], "warmup": 0,
        "warmup_note": "no warm-up timestep: compiled C++ with no JIT or caches to prime; the untimed setup "
                       "(assembly + Schur context) touches the whole working set first",
        "ms_per_step": 1e3 * r["seconds"] / r["steps"], "higher_is_better": True,
        "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded IC u0 = m + 0.01 U(-1,1), SURVEY.md 8(d); no dataset involved)",
        "parallelism": f"{procs} concurrent single-threaded instances on the host CPU",
        "cpu_baseline": {"value": r["value"], "unit": "DoF/s", "cores": procs, "kind": r["kind"], "sample": sample},
        "e2e": {"value": r["value"], "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gmres_iters": r["gmres_iters"], "setup_s": r["setup_s"],
    })
    if single is not None:
        line["single_instance"] = {
            "value": single["value"], "unit": "DoF/s", "cores": 1, "steps": single["steps"],
            "seconds": single["seconds"], "setup_s": single["setup_s"], "gmres_iters": single["gmres_iters"],
            "sample": "one instance alone on the idle host (one core), same workload and timing as above"}
    print(json.dumps(line), flush=True)
    return 0


# in-step kernel timing: the fine-level launch of each okg_kernel_timing id, matched by
# kernel template (demangled name prefix) and the largest grid of that template
def _kt_prefixes(dim):
    t = f"okg::k_tiled<{dim}, "
    return {"smooth": t + "0, 2,", "resid": t + "0, 1,", "pre2": t + "1, 2,", "post_acc": t + "0, 4,",
            "cheb": t + "0, 5,", "jacobian": f"okg::k_tiled_c<{dim}, 5,", "restrict": f"okg::k_restrict<{dim}>",
            "prolong": t + "2, 2,"}


def instep_profile(ctx, torch):
    """CUPTI activity records (torch.profiler/kineto) of ONE extra timestep after the
    timed region: per (kernel, grid) the launch count and device time."""
    import tempfile
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ctx.step_resident()
        torch.cuda.synchronize()
    fd, path = tempfile.mkstemp(suffix=".json")
    os.close(fd)
    try:
        prof.export_chrome_trace(path)
        tr = json.load(open(path))
    finally:
        os.unlink(path)
    agg, total = {}, 0.0
    for ev in tr.get("traceEvents", []):
        if ev.get("cat") != "kernel":
            continue
        grid = tuple(ev.get("args", {}).get("grid", (0, 0, 0)))
        d = agg.setdefault((ev["name"], grid), {"n": 0, "us": 0.0})
        d["n"] += 1
        d["us"] += float(ev.get("dur", 0.0))
        total += float(ev.get("dur", 0.0))
    return agg, total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="okg", choices=["okg", "reference"])
    ap.add_argument("--workload", default="c4_3d128", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of reference CPU work (cpu_baseline)")
    ap.add_argument("--ref-budget", type=float, default=60.0,
                    help="--impl reference: seconds of timed newton_solve per instance (at least one timestep)")
    ap.add_argument("--ref-procs", type=int, default=0, help="--impl reference: concurrent instances (0: auto)")
    ap.add_argument("--ref-no-single", action="store_true", help="--impl reference: skip the one-instance run")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="N > 1: weak = mesh grows with N (WEAK_N), strong = the workload's mesh split N ways "
                         "(default per workload: configs[3] strong, configs[4] weak)")
    ap.add_argument("--no-kernels", action="store_true", help="skip the per-kernel timings")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.scaling is None:
        args.scaling = DEFAULT_SCALING.get(args.workload, "strong")

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (127.0.0.1 rendezvous)
        if args.impl != "reference":
            import torch
            have = torch.cuda.device_count()
            if have < args.gpus:
                raise SystemExit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs on this node, found {have}")
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU "
                         f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus")
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (rank / nranks) on stderr
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    device = local_rank if world > 1 else 0

    import paper_1603_04570_b200 as okg
    from paper_1603_04570_b200 import _lib
    import ctypes as C

    _, _, eps, m, seed, n_cpu, desc = WORKLOADS[args.workload]
    dim, n = workload_mesh(args.workload, world, args.scaling)
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
        print(f"okg: rank {rank} of nranks {world}: solver NCCL communicator initialised on cuda:{device}, "
              f"x-planes per rank {ctx.slab_planes}", file=sys.stderr, flush=True)
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

    # ---- per-kernel timing: in-step (CUPTI) and alone L2-cold (CUDA events) ----
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        try:
            peak = float(json.load(open(peaks_path))["hbm_gbs"])
            peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)"
        except Exception:
            pass
    kernels, roofline, step_kernel_us = {}, None, None
    if not args.no_kernels:
        try:
            ctx.set_state(ic)
            agg, step_kernel_us = instep_profile(ctx, torch)
        except Exception as e:  # report, never fail the GPU line
            agg, step_kernel_us = {}, None
            print(f"bench.py: in-step profile failed: {e}", file=sys.stderr)
        pre = _kt_prefixes(dim)
        ctx.linearize(u0)
        for kid, name in enumerate(_lib.KT_NAMES):
            ms, by = C.c_double(), C.c_double()
            ent = {}
            if _lib.lib.okg_kernel_timing_ex(ctx.handle, kid, 20, _lib.KT_COLD | _lib.KT_NO_PDL,
                                             C.byref(ms), C.byref(by)) == 0:
                ent = {"alg_bytes": by.value, "cold_us": ms.value * 1e3,
                       "cold_gbs": by.value / (ms.value * 1e-3) / 1e9}
            cand = [(k, d) for k, d in agg.items() if k[0].startswith("void " + pre[name])]
            if cand and ent:
                (kname, grid), d = max(cand, key=lambda kd: kd[0][1][0] * kd[0][1][1] * kd[0][1][2])
                avg = d["us"] / d["n"]
                if name == "cheb":
                    # in the step every other Chebyshev step leaves x alone (16 of its 48 B/vertex
                    # less, okg_host.cu cheb()): the in-step mean is over both kinds of step
                    k = cfg.cheby_iters
                    nskip = sum(1 for j in range(1, k - 1) if (j & 1) and j != k - 2)
                    ent["alg_bytes_instep_mean"] = ent["alg_bytes"] * (48.0 * (k - 1) - 16.0 * nskip) / (48.0 * (k - 1))
                ent.update({"kernel": kname.split("(")[0].replace("void ", ""), "grid": list(grid),
                            "instep_n": d["n"], "instep_us": avg,
                            "instep_gbs": ent.get("alg_bytes_instep_mean", ent["alg_bytes"]) / (avg * 1e-6) / 1e9,
                            "share_of_step": d["us"] / step_kernel_us if step_kernel_us else None})
            if ent:
                kernels[name] = ent
        ctx.clear_linearization()
        ranked = sorted((k for k in kernels if "share_of_step" in kernels[k]),
                        key=lambda k: -kernels[k]["share_of_step"])
        if ranked:
            dom, d = ranked[0], kernels[ranked[0]]
            roofline = {"bound": "hbm", "kernel": f"{dom} ({d['kernel']}, grid {d['grid'][0]})",
                        "achieved": d["instep_gbs"], "peak": peak, "unit": "GB/s", "frac": d["instep_gbs"] / peak,
                        "peak_source": peak_src, "traffic": None,
                        "timing": ("in-step: mean device time of this kernel's launches during one timestep "
                                   "(CUPTI activity records via torch.profiler, one extra step after the "
                                   "timed region); cold_us = alone, L2 flushed before every launch, no PDL"),
                        "alg_bytes_per_launch": d.get("alg_bytes_instep_mean", d["alg_bytes"]),
                        "avg_launch_us": d["instep_us"],
                        "share_of_step": d["share_of_step"], "cold_us": d["cold_us"],
                        "cold_frac": d["cold_gbs"] / peak}
            if roofline["frac"] > 1.0:
                roofline["note"] = ("in-step time above the measured copy peak: part of this kernel's operands "
                                    "(written by the previous kernels of the step) is still in the 126 MB L2; "
                                    "cold_frac is the HBM-only figure")
            prof = os.path.join(ROOT, "profiles", "traffic.json")
            if os.path.exists(prof):
                try:
                    tr = json.load(open(prof)).get(args.workload, {}).get(dom)
                    if tr:
                        roofline["traffic"] = tr
                except Exception:
                    pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = ref_instance((dim, n_cpu, eps, m, seed, 500, args.cpu_budget, 100))
            cpu = {"value": r["value"], "unit": "DoF/s", "cores": 1, "kind": r["kind"],
                   "sample": (f"reduced size: {dim}D {n_cpu}^{dim} ({r['N']} vertices; the workload's own "
                              f"{n}^{dim} needs minutes of reference setup + solve per timestep, timed by "
                              f"bench.py --impl reference), same parameters and seeded IC, the first "
                              f"{r['steps']} timesteps of the reference newton_solve on one host core, timed "
                              f"by its own stats.seconds; CPU {_cpu_model()}, nproc {os.cpu_count()}")}
        except Exception as e:  # report, never fail the GPU line
            cpu = {"value": None, "unit": "DoF/s", "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded IC u0 = m + 0.01 U(-1,1), SURVEY.md 8(d); no dataset involved)",
            "config": workload_config(args.workload, dim, n),
            "parallelism": "1 GPU" if world == 1 else
                           (f"{world} x-plane slabs, one per GPU/process; ghost planes by NCCL send/recv, "
                            f"Krylov sums by NCCL allreduce; planes per rank {ctx.slab_planes}"),
            "setup_s": setup_s, "levels": ctx.level_sizes,
            "newton_iters": [s.newton_iters for s in stats],
            "gmres_iters": [s.gmres_iters for s in stats],
            "clocks": clocks_info,
            "e2e": {"value": e2e_value, "unit": "DoF/s", "h2d_bytes_per_step": 2 * N * 8,
                    "d2h_bytes_per_step": 2 * N * 8},
            "gpu_launches": launches,
            "roofline": roofline,
            "kernels": kernels,
            "step_kernel_us": step_kernel_us,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
