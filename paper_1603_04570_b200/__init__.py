"""B200-native Newton linear solve of the theta-method P1 Ohta-Kawasaki system.

Host-side mirror of the reference okflow API for the Newton-solve path
(/root/reference/proj/include/okflow: params.hpp, mesh.hpp, precond.hpp,
krylov.hpp, model.hpp), driving the sm_100a kernels of ``libokg.so``
through the C ABI in ``include/okg.h``.  Same names, argument meaning and
error behaviour as the reference:

    cfg = SolverConfig(dim=3, n=128, m=0.0, dt=4e-4, gmres_tol=1e-10, gmres_restart=30)
    mesh = build_mesh(cfg.dim, cfg.n)                       # mesh.hpp:87
    ctx = make_schur_context(mesh, cfg)                     # precond.hpp:126
    state = State(u=seeded_ic(mesh.num_vertices(), 2, 0.0), w=np.zeros(...))
    next_state, stats = newton_solve(state, mesh, ctx, cfg) # model.hpp:165

All arithmetic runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Tuple

import numpy as np

from . import _lib
from ._lib import (CannotCoarsen, ConfigError, CudaError, InconsistentState, InvalidArgument,  # noqa: F401
                   NumericalError, OkgError, check, lib)

__all__ = [
    "SolverConfig", "StructuredMesh", "build_mesh", "State", "IterationStats", "KrylovResult",
    "SchurContext", "make_schur_context", "compute_c", "residual", "newton_solve", "advance",
    "run_steps", "apply_block", "jacobian_operator", "block_preconditioner", "LinearOperator",
    "gmres", "seeded_ic", "DeviceArray", "total_mass", "energy", "integrate_double_well",
    "initial_state", "run_simulation", "SimulationResult",
    "InvalidArgument", "NumericalError", "ConfigError", "InconsistentState", "CannotCoarsen",
    "CudaError", "OkgError",
]


# --------------------------------------------------------------------------------------
# params.hpp:14-117
# --------------------------------------------------------------------------------------
@dataclass
class SolverConfig:
    eps: float = 0.02
    sigma: float = 100.0
    m: float = 0.4
    theta: float = 0.5
    dt: float = 4.0e-4
    n_steps: int = 25
    dim: int = 2
    n: int = 64
    newton_tol: float = 1e-8
    newton_maxit: int = 20
    gmres_tol: float = 1e-6
    gmres_maxit: int = 200
    gmres_restart: int = 0
    cheby_iters: int = 10
    cheby_precond: str = "jacobi"
    richardson_steps: int = 2
    mg_cycles: int = 5
    mg_pre: int = 2
    mg_post: int = 2
    mg_omega: float = 2.0 / 3.0
    min_coarse_size: int = 500
    threads: int = 1
    max_dofs: int = 2000000
    mesh_study_n: List[int] = field(default_factory=lambda: [32, 64, 128])
    eps_list: List[float] = field(default_factory=lambda: [0.02, 0.01])
    output_dir: str = "."
    snapshot_every: int = 0

    def num_vertices(self) -> int:
        s = self.n + 1
        return s ** self.dim

    def to_params(self, device: int = 0, shat_perturb: float = 0.0, use_graphs: bool = True,
                  tiled_min_n: int = 0, tail_max_vertices: int = 0, pdl: bool = True,
                  mg_fuse: int = 0, nslabs: int = 1, slab_devices: bool = False,
                  tail_cluster: int = 0, coarse_split: int = 0,
                  mg_collapse: int = 0, rep_max_vertices: int = 0) -> _lib.Params:
        p = _lib.Params()
        lib.okg_default_params(C.byref(p))
        for name in ("dim", "n", "eps", "sigma", "m", "theta", "dt", "newton_tol", "newton_maxit",
                     "gmres_tol", "gmres_maxit", "gmres_restart", "cheby_iters", "richardson_steps",
                     "mg_cycles", "mg_pre", "mg_post", "mg_omega", "min_coarse_size", "max_dofs"):
            setattr(p, name, getattr(self, name))
        p.shat_perturb = shat_perturb
        p.device = device
        p.use_graphs = 1 if use_graphs else 0
        p.tiled_min_n = tiled_min_n
        p.tail_max_vertices = tail_max_vertices
        p.disable_pdl = 0 if pdl else 1
        p.mg_fuse = mg_fuse
        p.nslabs = nslabs
        p.slab_devices = 1 if slab_devices else 0
        p.tail_cluster = tail_cluster
        p.coarse_split = coarse_split
        p.mg_collapse = mg_collapse
        p.rep_max_vertices = rep_max_vertices
        p.cheby_ssor = 1 if self.cheby_precond == "ssor" else 0
        return p

    def validate(self) -> None:
        """SolverConfig::validate (params.hpp:67-116): the first violated constraint, in
        the reference's order and with its message (ConfigError)."""
        def bad(msg):
            raise ConfigError("config: " + msg)
        if not self.eps > 0.0: bad("eps must be positive")
        if self.sigma < 0.0: bad("sigma must be nonnegative")
        if not abs(self.m) < 1.0: bad("mean m must satisfy |m| < 1")
        if not self.theta > 0.0 or self.theta > 1.0: bad("theta must lie in (0, 1]")
        if not self.dt > 0.0: bad("dt must be positive")
        if self.n_steps < 0: bad("n_steps must be nonnegative")
        if self.dim not in (2, 3): bad("dim must be 2 or 3")
        if self.n < 1: bad("n must be at least 1")
        if not self.newton_tol > 0.0: bad("newton_tol must be positive")
        if self.newton_maxit < 1: bad("newton_maxit must be at least 1")
        if not self.gmres_tol > 0.0: bad("gmres_tol must be positive")
        if self.gmres_maxit < 1: bad("gmres_maxit must be at least 1")
        if self.gmres_restart < 0: bad("gmres_restart must be nonnegative")
        if self.cheby_iters < 1: bad("cheby_iters must be at least 1")
        if self.cheby_precond not in ("jacobi", "ssor"): bad("cheby_precond must be 'jacobi' or 'ssor'")
        if self.richardson_steps < 1: bad("richardson_steps must be at least 1")
        if self.mg_cycles < 1: bad("mg_cycles must be at least 1")
        if self.mg_pre < 0 or self.mg_post < 0 or self.mg_pre + self.mg_post < 1:
            bad("need at least one smoothing sweep per cycle")
        if not self.mg_omega > 0.0 or not self.mg_omega < 2.0: bad("mg_omega must lie in (0, 2)")
        if self.min_coarse_size < 1: bad("min_coarse_size must be at least 1")
        if any(sn < 1 for sn in self.mesh_study_n): bad("mesh_study_n entries must be >= 1")
        if any(not se > 0.0 for se in self.eps_list): bad("eps_list entries must be positive")
        if self.threads < 1: bad("threads must be at least 1")
        if self.max_dofs < 1: bad("max_dofs must be at least 1")
        if self.snapshot_every < 0: bad("snapshot_every must be nonnegative")
        if self.num_vertices() > self.max_dofs:
            bad(f"mesh has {self.num_vertices()} vertices, exceeding max_dofs = {self.max_dofs}")
        # and the same checks through the C ABI (okg_validate_params) for the solver fields
        check(lib.okg_validate_params(C.byref(self.to_params())))


def compute_c(dt: float, theta: float, sigma: float) -> float:
    """precond.hpp:31-38."""
    if not dt > 0.0:
        raise InvalidArgument("compute_c: dt must be positive")
    if not theta > 0.0 or theta > 1.0:
        raise InvalidArgument("compute_c: theta must lie in (0, 1]")
    if sigma < 0.0:
        raise InvalidArgument("compute_c: sigma must be nonnegative")
    return dt * theta / (1.0 + dt * theta * sigma)


# --------------------------------------------------------------------------------------
# mesh.hpp:20-157 (arrays produced by libokg, bit-identical to build_mesh)
# --------------------------------------------------------------------------------------
@dataclass
class StructuredMesh:
    dim: int
    n: int
    h: float
    vertices: np.ndarray  # (N, dim)
    cells: np.ndarray     # (ncells, dim+1) int32

    def num_vertices(self) -> int:
        return self.vertices.shape[0]

    def num_cells(self) -> int:
        return self.cells.shape[0]

    def grid_index(self, i: int, j: int, k: int = 0) -> int:
        s = self.n + 1
        return i * s + j if self.dim == 2 else (i * s + j) * s + k

    def grid_coords(self, v: int):
        s = self.n + 1
        if self.dim == 2:
            return (v // s, v % s, 0)
        return (v // (s * s), (v // s) % s, v % s)


def build_mesh(dim: int, n: int, with_arrays: bool = True) -> StructuredMesh:
    if dim not in (2, 3):
        raise InvalidArgument("build_mesh: dim must be 2 or 3")
    if n < 1:
        raise InvalidArgument("build_mesh: n must be positive")
    s = n + 1
    nv = s ** dim
    if not with_arrays:
        return StructuredMesh(dim, n, 1.0 / n, np.empty((nv, 0)), np.empty((0, dim + 1), np.int32))
    ncell = 2 * n * n if dim == 2 else 6 * n ** 3
    v = np.empty((nv, dim))
    c = np.empty((ncell, dim + 1), dtype=np.int32)
    check(lib.okg_mesh(dim, n, v.ctypes.data_as(_lib._dp), c.ctypes.data_as(C.POINTER(C.c_int32))))
    return StructuredMesh(dim, n, 1.0 / n, v, c)


def nccl_unique_id() -> bytes:
    """The 128-byte NCCL id rank 0 makes for okg_create_rank (share it with every rank)."""
    buf = C.create_string_buffer(128)
    check(lib.okg_nccl_unique_id(buf, 128))
    return buf.raw


def slab_partition(dim: int, n: int, nslabs: int, rank: int, min_coarse_size: int = 500,
                   rep_max_vertices: int = 0):
    """The slab partition the contexts use (okg_slab_partition): returns
    (levels, rep_level, [(lo, hi) owned x-planes per level]).  rep_max_vertices as in
    okg_params (0 = default 3,000,000, < 0 = split as deep as 2 planes per slab)."""
    lv, rep = C.c_int32(), C.c_int32()
    lo = (C.c_int32 * 32)()
    hi = (C.c_int32 * 32)()
    check(lib.okg_slab_partition(dim, n, min_coarse_size, nslabs, rank, C.c_int64(rep_max_vertices),
                                 C.byref(lv), C.byref(rep), lo, hi))
    return lv.value, rep.value, [(lo[l], hi[l]) for l in range(lv.value)]


def seeded_ic(nverts: int, seed: int, m: float) -> np.ndarray:
    """Builder-defined seeded IC of SURVEY.md 8(d): u0 = m + 0.01*U(-1,1), splitmix64(seed, vertex)."""
    u = np.empty(nverts)
    check(lib.okg_seeded_ic(nverts, seed, m, u.ctypes.data_as(_lib._dp)))
    return u


# --------------------------------------------------------------------------------------
# model.hpp:25-42, krylov.hpp:21-28
# --------------------------------------------------------------------------------------
@dataclass
class State:
    u: np.ndarray
    w: np.ndarray
    t: float = 0.0
    step: int = 0


@dataclass
class IterationStats:
    step: int = 0
    t: float = 0.0
    newton_iters: int = 0
    gmres_iters: List[int] = field(default_factory=list)
    residual_norm: float = 0.0
    mass: float = 0.0
    energy: float = float("nan")  # filled by advance / run_simulation (okg_energy)
    seconds: float = 0.0
    converged: bool = True
    kernel_launches: int = 0


@dataclass
class KrylovResult:
    x: np.ndarray
    iterations: int
    residual_norms: List[float]
    converged: bool
    stagnated: bool
    final_residual: float


class DeviceArray:
    """A raw fp64 device buffer owned through the C ABI (no torch needed)."""

    def __init__(self, n: int, device: int = 0):
        self.n = int(n)
        self.ptr = C.c_void_p()
        check(lib.okg_device_alloc(device, max(self.n, 1) * 8, C.byref(self.ptr)))

    @classmethod
    def from_numpy(cls, a: np.ndarray, device: int = 0) -> "DeviceArray":
        a = np.ascontiguousarray(a, dtype=np.float64)
        d = cls(a.size, device)
        check(lib.okg_memcpy_h2d(d.ptr, a.ctypes.data_as(C.c_void_p), a.size * 8))
        return d

    @classmethod
    def view(cls, base: "DeviceArray", offset: int, n: int) -> "DeviceArray":
        """Non-owning view of base[offset : offset + n] (offset in doubles)."""
        if offset < 0 or offset + n > base.n:
            raise ValueError("DeviceArray.view: out of range")
        d = cls.__new__(cls)
        d.n = int(n)
        d.ptr = C.c_void_p(base.ptr.value + 8 * int(offset))
        d.base = base
        return d

    def numpy(self) -> np.ndarray:
        out = np.empty(self.n)
        check(lib.okg_memcpy_d2h(out.ctypes.data_as(C.c_void_p), self.ptr, self.n * 8))
        return out

    def free(self):
        if getattr(self, "base", None) is not None:  # a view owns nothing
            self.ptr = C.c_void_p()
            return
        if self.ptr:
            lib.okg_device_free(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# --------------------------------------------------------------------------------------
# precond.hpp:56-181 -- the context (plus the device workspace of the whole solve)
# --------------------------------------------------------------------------------------
class SchurContext:
    def __init__(self, cfg: SolverConfig, device: int = 0, shat_perturb: float = 0.0,
                 use_graphs: bool = True, tiled_min_n: int = 0, tail_max_vertices: int = 0,
                 pdl: bool = True, mg_fuse: int = 0, nslabs: int = 1, slab_devices: bool = False,
                 rank: Optional[int] = None, nranks: int = 1, nccl_id: Optional[bytes] = None,
                 tail_cluster: int = 0, coarse_split: int = 0, mg_collapse: int = 0,
                 rep_max_vertices: int = 0):
        """nslabs > 1: x-plane slab decomposition, one host thread + stream per
        slab, all on `device` (slab_devices=False, the 1-GPU emulation) or slab r on device
        `device + r`.  rank/nranks/nccl_id: one process per GPU (okg_create_rank), this
        process owning slab `rank`; host arrays stay full-size, the rank reads/writes its
        own planes."""
        self.cfg = cfg
        self.device = device
        self.handle = C.c_void_p()
        params = cfg.to_params(device, shat_perturb, use_graphs, tiled_min_n, tail_max_vertices, pdl, mg_fuse,
                               nslabs, slab_devices, tail_cluster, coarse_split, mg_collapse,
                               rep_max_vertices)
        if rank is None:
            check(lib.okg_create(C.byref(params), C.byref(self.handle)))
        else:
            idbuf = C.create_string_buffer(bytes(nccl_id), len(nccl_id)) if nccl_id is not None else None
            check(lib.okg_create_rank(C.byref(params), rank, nranks, idbuf, C.byref(self.handle)))
        self.rank = 0 if rank is None else rank
        info = _lib.Info()
        check(lib.okg_get_info(self.handle, C.byref(info)))
        self.info = info
        self.n = int(info.num_vertices)
        self.eps = cfg.eps
        self.c = info.c
        self.sqrt_c = info.sqrt_c
        self.a_coeff = info.a_coeff
        self.dt_theta = info.dt_theta
        self.lambda_lo = info.lambda_lo
        self.lambda_hi = info.lambda_hi
        self.eps_sqrt_c = info.eps_sqrt_c
        self.levels = int(info.levels)
        self.level_sizes = [int(info.level_size[i]) for i in range(self.levels)]
        self.level_n = [int(info.level_n[i]) for i in range(self.levels)]
        self.device_bytes = int(info.device_bytes)
        self.graph_nodes = int(info.graph_nodes)
        self.tail_start = int(info.tail_start)
        self.tail_cluster = int(info.tail_cluster)
        self.tiled_levels = [l for l in range(self.levels) if (info.tiled_mask >> l) & 1]
        self.coarse_rows = int(info.coarse_rows)
        self.collapse_level = int(info.collapse_level)
        self.nslabs = int(info.nslabs)
        self.rep_level = int(info.rep_level)
        self.slab_planes = [(int(info.slab_ilo[r]), int(info.slab_ihi[r])) for r in range(self.nslabs)]
        self.Me_set = False

    def rows(self) -> int:
        return self.n

    def close(self):
        if self.handle:
            lib.okg_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- per-operator entry points (host arrays in/out) ----
    def _out_size(self, kind: int, level: int) -> int:
        if kind in (_lib.OP_SHAT, _lib.OP_PROLONG, _lib.OP_VCYCLE):
            return self.level_sizes[level]
        if kind == _lib.OP_RESTRICT:
            return self.level_sizes[level + 1]
        if kind in (_lib.OP_BLOCK, _lib.OP_JACOBIAN):
            return 2 * self.n
        if kind == _lib.OP_COARSE_SOLVE:
            return self.level_sizes[-1]
        return self.n

    def apply_dev(self, kind: int, x: DeviceArray, y: DeviceArray, level: int = 0):
        check(lib.okg_apply(self.handle, kind, level, x.ptr, y.ptr))

    def apply(self, kind: int, x: np.ndarray, level: int = 0) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self._out_size(kind, level))
        check(lib.okg_apply_host_n(self.handle, kind, level, x.ctypes.data_as(_lib._dp), x.size,
                                   y.ctypes.data_as(_lib._dp), y.size))
        return y

    def linearize(self, u: np.ndarray):
        """ctx.Me = assemble_coefficient_mass(mesh, u)  (model.hpp:184-185)."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        check(lib.okg_linearize_host_n(self.handle, u.ctypes.data_as(_lib._dp), u.size))
        self.Me_set = True

    def linearize_dev(self, u: DeviceArray):
        check(lib.okg_linearize(self.handle, u.ptr))
        self.Me_set = True

    def clear_linearization(self):
        check(lib.okg_clear_linearization(self.handle))
        self.Me_set = False

    def residual(self, nxt: State, old: State) -> Tuple[np.ndarray, np.ndarray]:
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (nxt.u, nxt.w, old.u, old.w)]
        if any(a.size != arrs[0].size for a in arrs):
            raise InvalidArgument("residual: states do not match the mesh")
        r1 = np.empty(self.n)
        r2 = np.empty(self.n)
        check(lib.okg_residual_host_n(self.handle, *[a.ctypes.data_as(_lib._dp) for a in arrs], arrs[0].size,
                                    r1.ctypes.data_as(_lib._dp), r2.ctypes.data_as(_lib._dp)))
        return r1, r2

    def gmres(self, b: np.ndarray, rel_tol: float, max_iter: int, restart: int = 0) -> KrylovResult:
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(2 * self.n)
        ks = _lib.KrylovStats()
        check(lib.okg_gmres_host_n(self.handle, b.ctypes.data_as(_lib._dp), x.ctypes.data_as(_lib._dp), b.size, rel_tol,
                                 max_iter, restart, C.byref(ks)))
        nn = min(ks.n_residual_norms, 512)
        return KrylovResult(x, ks.iterations, list(ks.residual_norms[:nn]), bool(ks.converged),
                            bool(ks.stagnated), ks.final_residual)

    def jacobi_spectrum(self) -> Tuple[float, float]:
        lo, hi = C.c_double(), C.c_double()
        check(lib.okg_jacobi_spectrum(self.handle, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    # ---- time level held on the device ----
    def set_state(self, s: State):
        u = np.ascontiguousarray(s.u, dtype=np.float64)
        w = np.ascontiguousarray(s.w, dtype=np.float64)
        if u.size != self.n or w.size != self.n:
            raise InvalidArgument("residual: states do not match the mesh")
        check(lib.okg_set_state(self.handle, u.ctypes.data_as(_lib._dp), w.ctypes.data_as(_lib._dp),
                                s.t, s.step))

    def get_state(self) -> State:
        u = np.empty(self.n)
        w = np.empty(self.n)
        t = C.c_double()
        st = C.c_int32()
        check(lib.okg_get_state(self.handle, u.ctypes.data_as(_lib._dp), w.ctypes.data_as(_lib._dp),
                                C.byref(t), C.byref(st)))
        return State(u, w, t.value, st.value)

    def step_resident(self) -> IterationStats:
        """newton_solve on the device-resident state; the context state advances."""
        ss = _lib.StepStats()
        check(lib.okg_newton_step(self.handle, C.byref(ss)))
        return _stats(ss)

    def advance_resident(self, with_energy: bool = True) -> IterationStats:
        """advance (model.hpp:218-227): newton_solve + mass (+ energy) of the new state."""
        ss = _lib.StepStats()
        check(lib.okg_advance(self.handle, 1 if with_energy else 0, C.byref(ss)))
        return _stats(ss)

    # ---- diagnostics (model.hpp:46-114); u=None: the device-resident state ----
    def _u_arg(self, u):
        if u is None:
            return None, None
        a = np.ascontiguousarray(u, dtype=np.float64)
        if a.size != self.n:
            raise InvalidArgument("energy: vector length mismatch")
        return a, a.ctypes.data_as(_lib._dp)

    def total_mass(self, u: Optional[np.ndarray] = None) -> float:
        keep, p = self._u_arg(u)
        out = C.c_double()
        check(lib.okg_total_mass(self.handle, p, C.byref(out)))
        return out.value

    def double_well(self, u: Optional[np.ndarray] = None) -> float:
        keep, p = self._u_arg(u)
        out = C.c_double()
        check(lib.okg_double_well(self.handle, p, C.byref(out)))
        return out.value

    def energy(self, u: Optional[np.ndarray] = None) -> Tuple[float, int]:
        """-> (energy, CG iterations of the potential solve)."""
        keep, p = self._u_arg(u)
        out, it = C.c_double(), C.c_int32()
        check(lib.okg_energy(self.handle, p, C.byref(out), C.byref(it)))
        return out.value, it.value

    def initial_state(self) -> Tuple[State, int]:
        """initial_state (model.hpp:93-114) into the context; -> (state, CG iterations)."""
        it = C.c_int32()
        check(lib.okg_initial_state(self.handle, C.byref(it)))
        return self.get_state(), it.value


def _stats(ss: "_lib.StepStats") -> IterationStats:
    ni = ss.newton_iters
    return IterationStats(step=ss.step, t=ss.t, newton_iters=ni,
                          gmres_iters=[int(ss.gmres_iters[i]) for i in range(min(ni, _lib.OKG_MAX_NEWTON))],
                          residual_norm=ss.residual_norm, seconds=ss.seconds,
                          converged=bool(ss.converged), kernel_launches=int(ss.kernel_launches),
                          mass=float(ss.mass), energy=float(ss.energy))


def make_schur_context(mesh: StructuredMesh, cfg: SolverConfig, shat_perturb: float = 0.0,
                       device: int = 0, use_graphs: bool = True) -> SchurContext:
    """precond.hpp:126-181 (M and K are implicit in the structured mesh)."""
    if mesh.dim != cfg.dim or mesh.n != cfg.n:
        raise InvalidArgument("schur context: operator size does not match mesh")
    return SchurContext(cfg, device=device, shat_perturb=shat_perturb, use_graphs=use_graphs)


# --------------------------------------------------------------------------------------
# operator.hpp:16-37 and precond.hpp:257-307
# --------------------------------------------------------------------------------------
@dataclass
class LinearOperator:
    n: int
    n_in: int
    apply_fn: Callable[[np.ndarray], np.ndarray]
    label: str = ""

    def rows(self) -> int:
        return self.n

    def cols(self) -> int:
        return self.n_in if self.n_in > 0 else self.n

    def apply(self, x: np.ndarray) -> np.ndarray:
        if np.asarray(x).size != self.cols():
            raise InvalidArgument(f"operator '{self.label}': input dimension mismatch")
        return self.apply_fn(x)

    __call__ = apply


def apply_block(ctx: SchurContext, r: np.ndarray) -> np.ndarray:
    if np.asarray(r).size != 2 * ctx.n:
        raise InvalidArgument("block preconditioner: stacked size mismatch")
    return ctx.apply(_lib.OP_BLOCK, r)


def jacobian_operator(ctx: SchurContext) -> LinearOperator:
    return LinearOperator(2 * ctx.n, 2 * ctx.n, lambda x: ctx.apply(_lib.OP_JACOBIAN, x), "coupled-jacobian")


def block_preconditioner(ctx: SchurContext) -> LinearOperator:
    return LinearOperator(2 * ctx.n, 2 * ctx.n, lambda r: apply_block(ctx, r), "block-triangular")


def gmres(ctx: SchurContext, b: np.ndarray, rel_tol: float, max_iter: int, restart: int = 0) -> KrylovResult:
    """gmres(jacobian_operator(ctx), block_preconditioner(ctx), b, ...) -- krylov.hpp:44."""
    return ctx.gmres(b, rel_tol, max_iter, restart)


# --------------------------------------------------------------------------------------
# model.hpp:46-279
# --------------------------------------------------------------------------------------
def residual(nxt: State, old: State, mesh: StructuredMesh, ctx: SchurContext, cfg: Optional[SolverConfig] = None):
    """model.hpp:121-148 -> (R1, R2)."""
    if len(nxt.u) != len(old.u) or len(nxt.w) != len(old.w) or len(nxt.u) != mesh.num_vertices():
        raise InvalidArgument("residual: states do not match the mesh")
    return ctx.residual(nxt, old)


def newton_solve(old: State, mesh: StructuredMesh, ctx: SchurContext,
                 cfg: Optional[SolverConfig] = None) -> Tuple[State, IterationStats]:
    """model.hpp:165-215: one implicit step; non-convergence is reported, not raised."""
    if len(old.u) != mesh.num_vertices():
        raise InvalidArgument("residual: states do not match the mesh")
    ctx.set_state(old)
    stats = ctx.step_resident()
    return ctx.get_state(), stats


def total_mass(mesh: StructuredMesh, ctx: SchurContext, u: np.ndarray) -> float:
    """model.hpp:46-48: b^T u (okg_total_mass)."""
    return ctx.total_mass(u)


def integrate_double_well(mesh: StructuredMesh, ctx: SchurContext, u: np.ndarray) -> float:
    """assembly.hpp:220-245 (okg_double_well)."""
    return ctx.double_well(u)


def energy(mesh: StructuredMesh, ctx: SchurContext, u: np.ndarray, cfg: Optional[SolverConfig] = None) -> float:
    """model.hpp:56-86 (okg_energy): raises InconsistentState / NumericalError like the reference."""
    if len(u) != mesh.num_vertices():
        raise InvalidArgument("energy: vector length mismatch")
    return ctx.energy(u)[0]


def initial_state(mesh: StructuredMesh, ctx: SchurContext, cfg: Optional[SolverConfig] = None) -> State:
    """model.hpp:93-114 (okg_initial_state)."""
    return ctx.initial_state()[0]


def advance(state: State, mesh: StructuredMesh, ctx: SchurContext,
            cfg: Optional[SolverConfig] = None) -> Tuple[State, IterationStats]:
    """model.hpp:218-227: newton_solve + mass + energy of the new state."""
    if len(state.u) != mesh.num_vertices():
        raise InvalidArgument("residual: states do not match the mesh")
    ctx.set_state(state)
    stats = ctx.advance_resident(True)
    return ctx.get_state(), stats


@dataclass
class SimulationResult:
    mesh: StructuredMesh
    stats: List[IterationStats]
    final_state: State


def run_simulation(cfg: SolverConfig, on_state: Optional[Callable[[StructuredMesh, State], None]] = None,
                   shat_perturb: float = 0.0, on_stats: Optional[Callable[[IterationStats], None]] = None,
                   ctx: Optional[SchurContext] = None, with_energy: bool = True) -> SimulationResult:
    """run_simulation (model.hpp:243-279): initial_state, then cfg.n_steps advances, all
    device-resident; the state leaves the GPU only for `on_state` observers."""
    cfg.validate()
    mesh = build_mesh(cfg.dim, cfg.n, with_arrays=False)
    own = ctx is None
    if own:
        ctx = make_schur_context(mesh, cfg, shat_perturb)
    try:
        state, _ = ctx.initial_state()
        init = IterationStats(step=0, t=0.0, mass=ctx.total_mass(), energy=ctx.energy()[0] if with_energy else float("nan"))
        stats = [init]
        if on_stats:
            on_stats(init)
        if on_state:
            on_state(mesh, state)
        for _ in range(cfg.n_steps):
            st = ctx.advance_resident(with_energy)
            stats.append(st)
            if on_stats:
                on_stats(st)
            if not st.converged:
                raise NumericalError(f"run_simulation: nonlinear solve failed at step {st.step} "
                                     f"(residual {st.residual_norm})")
            if on_state:
                on_state(mesh, ctx.get_state())
        return SimulationResult(mesh, stats, ctx.get_state())
    finally:
        if own:
            ctx.close()


def run_steps(ctx: SchurContext, state: State, n_steps: int,
              on_stats: Optional[Callable[[IterationStats], None]] = None) -> Tuple[State, List[IterationStats]]:
    """The timestep loop of run_simulation (model.hpp:266-276), device-resident between steps."""
    ctx.set_state(state)
    out = []
    for _ in range(n_steps):
        st = ctx.step_resident()
        out.append(st)
        if on_stats:
            on_stats(st)
        if not st.converged:
            raise NumericalError(f"run_simulation: nonlinear solve failed at step {st.step} "
                                 f"(residual {st.residual_norm})")
    return ctx.get_state(), out
