"""Per-timestep reference fixtures at the BASELINE.json sizes -- TEST INFRASTRUCTURE.

Runs the UNMODIFIED reference (oracle/_ref/libokref.so: the okflow headers compiled
by oracle/Makefile) through newton_solve (/root/reference/proj/include/okflow/model.hpp:165-215)
for every timestep of BASELINE configs[1]-[3] and records, per timestep:

  newton_iters, gmres_iters[newton], residual_norm, seconds (stats.seconds),
  ||u||, ||w|| and 64 Rademacher projections of u and w (tests/sketch.py),

plus the full u/w fields for the 2D meshes <= 256^2 (every step) and 512^2 (last
step).  tests/test_gpu_baseline_full.py replays the same timesteps on the GPU and
checks counts within +-1 and the estimated relative l2 of u and w <= 1e-8.

Settings (BASELINE.json / SURVEY.md 8(d)): sigma = 100, theta = 0.5, dt = eps^2,
GMRES(30) rtol 1e-10, newton_tol 1e-8, seeded IC u0 = m + 0.01 U(-1,1) (SURVEY 8(d)
splitmix64), w0 = 0.  The reference needs ~30 min (3D 128^3, 10 steps) of one core;
run the cases as parallel processes:

    make -C oracle ref
    python tests/golden/make_baseline_fixtures.py            # all cases, one process each
    python tests/golden/make_baseline_fixtures.py c2_n256    # one case
"""
import os
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
OUT = os.path.join(HERE, "baseline")

# name: (dim, n, eps, m, seed, steps, full-field steps)
CASES = {
    # configs[1]: 2D mesh-independence sweep, 5 timesteps (seed not stated: 0)
    "c2_n128": (2, 128, 0.02, 0.0, 0, 5, "all"),
    "c2_n256": (2, 256, 0.02, 0.0, 0, 5, "all"),
    "c2_n512": (2, 512, 0.02, 0.0, 0, 5, "last"),
    "c2_n1024": (2, 1024, 0.02, 0.0, 0, 5, None),
    "c2_n2048": (2, 2048, 0.02, 0.0, 0, 5, None),
    # configs[2]: eps-robustness sweep at 1024^2, m = 0.1, seed 1, 10 timesteps
    "c3_e040": (2, 1024, 0.04, 0.1, 1, 10, None),
    "c3_e020": (2, 1024, 0.02, 0.1, 1, 10, None),
    "c3_e010": (2, 1024, 0.01, 0.1, 1, 10, None),
    "c3_e005": (2, 1024, 0.005, 0.1, 1, 10, None),
    # configs[3]: 3D 128^3, seed 2, 10 timesteps
    "c4_3d128": (3, 128, 0.02, 0.0, 2, 10, None),
}


def make(name):
    import pyoracle as po
    from sketch import sketch

    dim, n, eps, m, seed, steps, full = CASES[name]
    t0 = time.time()
    p = po.baseline_params(dim, n, eps=eps, m=m, kind="ref")
    o = po.Oracle(p, "ref")
    setup_s = time.time() - t0
    N = o.n
    u = po.seeded_ic(N, seed, m, "ref")
    w = np.zeros(N)
    rec = {k: [] for k in ("newton_iters", "gmres_iters", "residual_norm", "seconds", "converged",
                           "norm_u", "norm_w", "proj_u", "proj_w")}
    fields = {}
    for step in range(steps):
        u, w, st = o.newton_solve(u, w)
        sk = sketch(u, w)
        rec["newton_iters"].append(st.newton_iters)
        gi = np.full(8, -1, dtype=np.int32)
        gi[: len(st.gmres_iters)] = st.gmres_iters
        rec["gmres_iters"].append(gi)
        rec["residual_norm"].append(st.residual_norm)
        rec["seconds"].append(st.seconds)
        rec["converged"].append(st.converged)
        for k in ("norm_u", "norm_w", "proj_u", "proj_w"):
            rec[k].append(sk[k])
        if full == "all" or (full == "last" and step == steps - 1):
            fields[f"u{step + 1}"] = u.copy()
            fields[f"w{step + 1}"] = w.copy()
        print(f"{name} step {step + 1}/{steps}: newton {st.newton_iters} gmres {st.gmres_iters} "
              f"{st.seconds:.1f}s", flush=True)
    o.close()
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(
        os.path.join(OUT, name + ".npz"),
        dim=dim, n=n, eps=eps, m=m, seed=seed, steps=steps, N=N, setup_s=setup_s,
        **{k: np.asarray(v) for k, v in rec.items()}, **fields)


def main(argv):
    names = argv or list(CASES)
    if len(names) == 1:
        make(names[0])
        return
    procs = {nm: subprocess.Popen([sys.executable, __file__, nm],
                                  stdout=open(os.path.join("/tmp", f"fix_{nm}.log"), "w"),
                                  stderr=subprocess.STDOUT) for nm in names}
    bad = [nm for nm, pr in procs.items() if pr.wait() != 0]
    if bad:
        raise SystemExit(f"failed: {bad} (logs in /tmp/fix_*.log)")


if __name__ == "__main__":
    main(sys.argv[1:])
