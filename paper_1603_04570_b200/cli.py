"""The reference's INI front end, study drivers and command line over the B200
solver.

  RunManifest, parse_config       config.hpp:18-236  (same keys, defaults and errors;
                                                      numbers through libc strtod/strtol
                                                      exactly like the reference)
  cmd_run                         driver.hpp:79-125  (io.cmd_run)
  cmd_mesh_study, cmd_eps_study   driver.hpp:127-205 (same CSV files and tables)
  main                            tools/okflow.cpp   (subcommands run | mesh-study |
                                                      eps-study | verify, --config,
                                                      --output, --threads, --perturb-shat;
                                                      exit 2 on a config error)

`verify` (dense spectral desk checks) is out of scope for the GPU path.
Usage: python -m paper_1603_04570_b200 run --config problem.ini
"""
from __future__ import annotations

import argparse
import ctypes as C
import dataclasses
import math
import os
import sys
from dataclasses import dataclass, field
from typing import List

from . import ConfigError, SolverConfig, run_simulation
from .io import cmd_run, format_g17

_libc = C.CDLL(None)
_libc.strtod.restype = C.c_double
_libc.strtod.argtypes = [C.c_char_p, C.POINTER(C.c_char_p)]
_libc.strtol.restype = C.c_long
_libc.strtol.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_int]


@dataclass
class RunManifest:
    config: SolverConfig = field(default_factory=SolverConfig)
    kind: str = "run"  # run | mesh-study | eps-study | verify
    shat_perturb: float = 0.0


def _trim(s: str) -> str:
    return s.strip(" \t\r\n")


def _strip_inline_comment(s: str) -> str:
    for i, ch in enumerate(s):
        if ch in "#;" and (i == 0 or s[i - 1] in " \t\n\v\f\r"):
            return s[:i]
    return s


def _strtod_full(v: str):
    b = v.encode()
    buf = C.create_string_buffer(b)
    end = C.c_char_p()
    x = _libc.strtod(buf, C.byref(end))
    consumed = C.cast(end, C.c_void_p).value - C.cast(buf, C.c_void_p).value
    return x, consumed == len(b)


def _strtol_full(v: str):
    b = v.encode()
    buf = C.create_string_buffer(b)
    end = C.c_char_p()
    x = _libc.strtol(buf, C.byref(end), 10)
    consumed = C.cast(end, C.c_void_p).value - C.cast(buf, C.c_void_p).value
    return x, consumed == len(b)


def _to_double(key: str, value: str) -> float:
    v = _trim(value)
    x, full = _strtod_full(v)
    if not v or not full:
        raise ConfigError(f"config: value for key '{key}' is not a number: '{value}'")
    return x


def _to_long(key: str, value: str) -> int:
    v = _trim(value)
    x, full = _strtol_full(v)
    if not v or not full:
        raise ConfigError(f"config: value for key '{key}' is not an integer: '{value}'")
    return x


def _to_int(key: str, value: str) -> int:
    x = _to_long(key, value)
    return ((x + 2 ** 31) % 2 ** 32) - 2 ** 31  # static_cast<int>(long)


def _to_list(key: str, value: str, conv) -> list:
    out = [conv(key, p) for p in (_trim(q) for q in value.split(",")) if p]
    if not out:
        raise ConfigError(f"config: value for key '{key}' is an empty list")
    return out


_SECTIONS = ("problem", "mesh", "solver", "output")
_KEYS = {
    "problem": {"eps": _to_double, "sigma": _to_double, "m": _to_double, "theta": _to_double,
                "eps_list": lambda k, v: _to_list(k, v, _to_double)},
    "mesh": {"dim": _to_int, "n": _to_int, "mesh_study_n": lambda k, v: _to_list(k, v, _to_int),
             "max_dofs": _to_long},
    "solver": {"dt": _to_double, "n_steps": _to_int, "newton_tol": _to_double, "newton_maxit": _to_int,
               "gmres_tol": _to_double, "gmres_maxit": _to_int, "gmres_restart": _to_int,
               "cheby_iters": _to_int, "cheby_precond": lambda k, v: v, "richardson_steps": _to_int,
               "mg_cycles": _to_int, "mg_pre": _to_int, "mg_post": _to_int, "mg_omega": _to_double,
               "min_coarse_size": _to_int, "threads": _to_int},
    "output": {"directory": lambda k, v: v, "snapshot_every": _to_int},
}
_FIELD = {"directory": "output_dir"}
_REQUIRED = ("eps", "sigma", "m", "theta", "dim", "n", "dt", "n_steps")


def parse_config(path: str) -> RunManifest:
    """config.hpp:114-236: the flat key = value format with sections [problem],
    [mesh], [solver], [output]; the returned manifest has passed validate()."""
    try:
        with open(path, "rb") as fh:
            raw = fh.read()
    except OSError:
        raise ConfigError(f"config: cannot open file: {path}")
    man = RunManifest()
    cfg = man.config
    seen = set()
    section = ""
    text = raw.decode("utf-8", errors="surrogateescape")
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines = lines[:-1]
    for lineno, line in enumerate(lines, start=1):
        t = _trim(_strip_inline_comment(_trim(line)))
        if not t:
            continue
        if t[0] == "[":
            if t[-1] != "]":
                raise ConfigError(f"config: malformed section header at line {lineno}: {t}")
            section = _trim(t[1:-1])
            if section not in _SECTIONS:
                raise ConfigError(f"config: unknown section [{section}]")
            continue
        eq = t.find("=")
        if eq < 0:
            raise ConfigError(f"config: expected key = value at line {lineno}: {t}")
        if not section:
            raise ConfigError(f"config: key outside any section at line {lineno}: {t}")
        key, value = _trim(t[:eq]), _trim(t[eq + 1:])
        if not key:
            raise ConfigError(f"config: empty key at line {lineno}")
        seen.add(key)
        conv = _KEYS[section].get(key)
        if conv is None:
            raise ConfigError(f"config: unknown key '{key}' in section [{section}] (line {lineno})")
        setattr(cfg, _FIELD.get(key, key), conv(key, value))
    for req in _REQUIRED:
        if req not in seen:
            raise ConfigError(f"config: missing required key: {req}")
    cfg.validate()
    return man


def _ensure_dir(cfg: SolverConfig) -> str:
    d = cfg.output_dir or "."
    try:
        os.makedirs(d, exist_ok=True)
    except OSError as e:
        raise ConfigError(f"output: cannot create directory '{d}': {e}") from e
    return d


def _avg_gmres_per_newton(stats) -> float:
    nw = sum(s.newton_iters for s in stats if s.step != 0)
    gm = sum(sum(s.gmres_iters) for s in stats if s.step != 0)
    return gm / nw if nw > 0 else 0.0


def _short(x: float) -> str:
    return "%.4g" % x


def cmd_mesh_study(man: RunManifest) -> int:
    """driver.hpp:127-156"""
    d = _ensure_dir(man.config)
    with open(os.path.join(d, "mesh_study.csv"), "w", newline="") as csv:
        csv.write("n,dofs,avg_gmres_per_newton\n")
        csv.flush()
        print(f"mesh study ({man.config.dim}D, eps = {_short(man.config.eps)})")
        print(f"{'n':>8}{'dofs':>12}{'avg GMRES per Newton':>24}")
        for n in man.config.mesh_study_n:
            cfg = dataclasses.replace(man.config, n=n)
            res = run_simulation(cfg, shat_perturb=man.shat_perturb)
            avg = _avg_gmres_per_newton(res.stats)
            dofs = 2 * cfg.num_vertices()
            csv.write(f"{n},{dofs},{format_g17(avg)}\n")
            csv.flush()
            print(f"{n:>8}{dofs:>12}{_short(avg):>24}")
    return 0


def cmd_eps_study(man: RunManifest) -> int:
    """driver.hpp:158-205: dx = eps/2 (n = round(2/eps)), dt = eps^2."""
    runs = []
    for eps in man.config.eps_list:
        n = int(math.floor(2.0 / eps + 0.5)) if 2.0 / eps >= 0 else int(math.ceil(2.0 / eps - 0.5))  # llround
        cfg = dataclasses.replace(man.config, eps=eps, n=n, dt=eps * eps)
        if cfg.num_vertices() > cfg.max_dofs:
            print(f"eps-study: refusing eps = {_short(eps)}: mesh n = {cfg.n} has {cfg.num_vertices()} "
                  f"vertices, exceeding max_dofs = {cfg.max_dofs}", file=sys.stderr)
            return 2
        runs.append(cfg)
    d = _ensure_dir(man.config)
    with open(os.path.join(d, "eps_study.csv"), "w", newline="") as csv:
        csv.write("eps,dx,dt,avg_gmres_per_newton\n")
        csv.flush()
        print(f"eps study ({man.config.dim}D)")
        print(f"{'eps':>12}{'dx':>12}{'dt':>14}{'avg GMRES per Newton':>24}")
        for cfg in runs:
            res = run_simulation(cfg, shat_perturb=man.shat_perturb)
            avg = _avg_gmres_per_newton(res.stats)
            dx = 1.0 / cfg.n
            csv.write(f"{format_g17(cfg.eps)},{format_g17(dx)},{format_g17(cfg.dt)},{format_g17(avg)}\n")
            csv.flush()
            print(f"{_short(cfg.eps):>12}{_short(dx):>12}{_short(cfg.dt):>14}{_short(avg):>24}")
    return 0


def run_manifest(man: RunManifest) -> int:
    if man.kind == "run":
        return cmd_run(man.config, man.config.output_dir, man.config.snapshot_every, man.shat_perturb)
    if man.kind == "mesh-study":
        return cmd_mesh_study(man)
    if man.kind == "eps-study":
        return cmd_eps_study(man)
    if man.kind == "verify":
        print("verify: the dense spectral desk checks are not part of the GPU path; run the reference's "
              "`okflow verify` (SURVEY 8: out of scope)", file=sys.stderr)
        return 1
    raise ConfigError(f"manifest: unknown kind '{man.kind}'")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="okflow-b200", description=(
        "Ohta-Kawasaki phase-field solver with a matched-product Schur block preconditioner "
        "(B200 Newton linear solve)"))
    sub = ap.add_subparsers(dest="kind", required=True)
    for name, desc in (("run", "time-step the configured problem, writing stats.csv and VTK snapshots"),
                       ("mesh-study", "repeat the run across the mesh list, writing mesh_study.csv"),
                       ("eps-study", "repeat the run across the eps list (dx = eps/2, dt = eps^2), "
                                     "writing eps_study.csv"),
                       ("verify", "spectral desk checks (reference only)")):
        p = sub.add_parser(name, help=desc)
        p.add_argument("--config", required=True, help="path to the configuration file")
        p.add_argument("--output", default="", help="output directory (overrides [output] directory)")
        p.add_argument("--threads", type=int, default=0, help="worker thread count (overrides [solver] threads)")
        p.add_argument("--perturb-shat", type=float, default=0.0,
                       help="fault injection: scale the shifted operator by 1+X (self-test)")
    a = ap.parse_args(argv)
    try:
        man = parse_config(a.config)
        man.kind = a.kind
        man.shat_perturb = a.perturb_shat
        if a.output:
            man.config.output_dir = a.output
        if a.threads > 0:
            man.config.threads = a.threads
        man.config.validate()
        return run_manifest(man)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 -- the reference's catch-all (tools/okflow.cpp)
        print(f"error: {e}", file=sys.stderr)
        return 1
