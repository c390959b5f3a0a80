"""Output formats of the reference over the B200 solver.

  format_g17   vtk.hpp:17-22      locale-independent, 17 significant digits, shortest form
  write_vtk    vtk.hpp:28-66      legacy-VTK STRUCTURED_POINTS, byte-identical to the reference
  cmd_run      driver.hpp:79-125  device-resident run streaming stats.csv; VTK snapshots are
                                  formatted and written by a background thread while the GPU
                                  computes the next steps
"""
from __future__ import annotations

import os
import sys
import threading
from typing import Optional

import numpy as np

from . import (NumericalError, ConfigError, InconsistentState, SchurContext, SolverConfig, State,
               run_simulation)


def format_g17(x: float) -> str:
    """C++ `os << std::setprecision(17) << x` under the classic locale == printf("%.17g")."""
    return "%.17g" % x


def _fmt_column(f: np.ndarray) -> str:
    return "\n".join("%.17g" % v for v in f.tolist()) + "\n"


def write_vtk(dim: int, n: int, u: np.ndarray, w: np.ndarray, path: str) -> None:
    s = n + 1
    nv = s ** dim
    if len(u) != nv or len(w) != nv:
        raise InconsistentState("write_vtk: field size does not match mesh")
    h = format_g17(1.0 / n)
    head = ("# vtk DataFile Version 3.0\nokflow state\nASCII\nDATASET STRUCTURED_POINTS\n"
            f"DIMENSIONS {s} {s} {s if dim == 3 else 1}\nORIGIN 0 0 0\nSPACING {h} {h} {h}\n"
            f"POINT_DATA {nv}\n")

    def native(f):  # reference index x slowest -> VTK x fastest (mesh.hpp:40-44)
        a = np.asarray(f, dtype=np.float64)
        return a.reshape((s, s, s) if dim == 3 else (s, s)).T.reshape(-1)

    body = ("SCALARS u double 1\nLOOKUP_TABLE default\n" + _fmt_column(native(u)) +
            "SCALARS w double 1\nLOOKUP_TABLE default\n" + _fmt_column(native(w)))
    try:
        with open(path, "wb") as fh:
            fh.write((head + body).encode("ascii"))
    except OSError as e:
        raise RuntimeError(f"write_vtk: cannot open {path}") from e


def stats_row(st) -> str:
    total = sum(st.gmres_iters)
    avg = total / st.newton_iters if st.newton_iters > 0 else 0.0
    return (f"{st.step},{st.newton_iters},{total},{format_g17(avg)},{format_g17(st.residual_norm)},"
            f"{format_g17(st.mass)},{format_g17(st.energy)},{format_g17(st.seconds)}\n")


STATS_HEADER = "step,newton_iters,total_gmres,avg_gmres,residual,mass,energy,seconds\n"


def cmd_run(cfg: SolverConfig, output_dir: str = ".", snapshot_every: int = 0, shat_perturb: float = 0.0,
            ctx: Optional[SchurContext] = None) -> int:
    """driver.hpp:79-125: returns 1 after a failed nonlinear solve (completed rows and
    snapshots stay on disk), else 0."""
    d = output_dir or "."
    try:
        os.makedirs(d, exist_ok=True)
    except OSError as e:
        raise ConfigError(f"output: cannot create directory '{d}': {e}") from e
    csv = open(os.path.join(d, "stats.csv"), "w", newline="")
    csv.write(STATS_HEADER)
    csv.flush()
    totals = [0, 0]
    pending: list = []

    def on_stats(st):
        if st.step == 0:
            return
        csv.write(stats_row(st))
        csv.flush()
        totals[0] += st.newton_iters
        totals[1] += sum(st.gmres_iters)

    def on_state(mesh, s: State):
        if not (s.step == 0 or (snapshot_every > 0 and s.step % snapshot_every == 0)):
            return
        for t in pending:
            t.join()
        pending.clear()
        path = os.path.join(d, f"state_{s.step}.vtk")
        t = threading.Thread(target=write_vtk, args=(cfg.dim, cfg.n, s.u.copy(), s.w.copy(), path))
        t.start()
        pending.append(t)

    try:
        run_simulation(cfg, on_state=on_state, shat_perturb=shat_perturb, on_stats=on_stats, ctx=ctx)
    except NumericalError as e:
        for t in pending:
            t.join()
        csv.close()
        print(f"run: {e}", file=sys.stderr)
        return 1
    for t in pending:
        t.join()
    csv.close()
    avg = totals[1] / totals[0] if totals[0] else 0.0
    print(f"run: {cfg.n_steps} steps, {cfg.dim}D n={cfg.n}, avg GMRES per Newton = {'%.4g' % avg}")
    return 0
