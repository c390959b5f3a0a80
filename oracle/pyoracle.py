"""ctypes binding of oracle/okoracle.h -- TEST INFRASTRUCTURE ONLY.

Loads either the reference compiled from /root/reference (``oracle/_ref/libokref.so``,
kind="ref") or the plain-C restatement (``oracle/libokport.so``, kind="port").
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` leg may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "ref": os.path.join(HERE, "_ref", "libokref.so"),
    "port": os.path.join(HERE, "libokport.so"),
}

M, K, A, SHAT, PROLONG, RESTRICT, VCYCLE, SHAT_INV, CHEB_M, CHEB_A = range(10)
ME, C_OP, SCHUR, SCHUR_TILDE_INV, S_INV_APPROX, BLOCK, JACOBIAN, NONLINEAR = range(10, 18)
COARSE_SOLVE = 18
SSOR_M = 19

ERRORS = {
    -1: ValueError,
    -2: ArithmeticError,
    -3: RuntimeError,
    -4: RuntimeError,
    -5: RuntimeError,
    -9: RuntimeError,
}
ERROR_NAMES = {-1: "invalid_argument", -2: "NumericalError", -3: "ConfigError",
               -4: "InconsistentState", -5: "CannotCoarsen", -9: "other"}


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERROR_NAMES.get(code, str(code))


class Params(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("n", C.c_int),
        ("eps", C.c_double), ("sigma", C.c_double), ("m", C.c_double),
        ("theta", C.c_double), ("dt", C.c_double),
        ("newton_tol", C.c_double), ("newton_maxit", C.c_int),
        ("gmres_tol", C.c_double), ("gmres_maxit", C.c_int), ("gmres_restart", C.c_int),
        ("cheby_iters", C.c_int), ("richardson_steps", C.c_int),
        ("mg_cycles", C.c_int), ("mg_pre", C.c_int), ("mg_post", C.c_int),
        ("mg_omega", C.c_double), ("min_coarse_size", C.c_int),
        ("shat_perturb", C.c_double), ("cheby_ssor", C.c_int),
    ]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_loaded = {}


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def load(kind: str = "ref"):
    if kind in _loaded:
        return _loaded[kind]
    lib = C.CDLL(LIBS[kind])
    lib.oko_create.restype = C.c_void_p
    lib.oko_create.argtypes = [C.POINTER(Params), _ip]
    lib.oko_destroy.argtypes = [C.c_void_p]
    lib.oko_last_error.restype = C.c_char_p
    lib.oko_num_vertices.restype = C.c_long
    lib.oko_num_vertices.argtypes = [C.c_void_p]
    lib.oko_levels.argtypes = [C.c_void_p]
    lib.oko_level_size.restype = C.c_long
    lib.oko_level_size.argtypes = [C.c_void_p, C.c_int]
    lib.oko_scalars.argtypes = [C.c_void_p, _dp]
    lib.oko_load_vector.argtypes = [C.c_void_p, _dp]
    lib.oko_level_dense.argtypes = [C.c_void_p, C.c_int, _dp]
    lib.oko_mesh.argtypes = [C.c_int, C.c_int, _dp, _ip]
    lib.oko_set_linearization.argtypes = [C.c_void_p, _dp]
    lib.oko_apply.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp]
    lib.oko_residual.argtypes = [C.c_void_p] + [_dp] * 6
    lib.oko_gmres.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int, C.c_int,
                              _ip, _dp, _ip, _ip, _dp, C.c_int, _ip]
    lib.oko_newton_solve.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _ip, _ip, _dp, _dp, _ip]
    lib.oko_jacobi_spectrum.argtypes = [C.c_void_p, _dp, _dp]
    lib.oko_seeded_ic.argtypes = [C.c_long, C.c_ulonglong, C.c_double, _dp]
    lib.oko_default_params.argtypes = [C.POINTER(Params)]
    lib.oko_total_mass.argtypes = [C.c_void_p, _dp, _dp]
    lib.oko_double_well.argtypes = [C.c_void_p, _dp, _dp]
    lib.oko_energy.argtypes = [C.c_void_p, _dp, _dp, _ip]
    lib.oko_initial_state.argtypes = [C.c_void_p, _dp, _dp, _ip]
    if kind == "ref":
        lib.oko_format_g17.argtypes = [C.c_double, C.c_char_p, C.c_int]
        lib.oko_write_vtk.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_char_p]
    _loaded[kind] = lib
    return lib


def _p(a):
    return a.ctypes.data_as(_dp)


def _check(lib, st):
    if st != 0:
        raise OracleError(st, lib.oko_last_error().decode())


def default_params(kind="ref", **kw) -> Params:
    lib = load(kind)
    p = Params()
    lib.oko_default_params(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def baseline_params(dim, n, eps=0.02, m=0.0, kind="ref", **kw) -> Params:
    """BASELINE.json settings: sigma=100, theta=.5, dt=eps^2, GMRES(30) rtol 1e-10."""
    base = dict(dim=dim, n=n, eps=eps, sigma=100.0, m=m, theta=0.5, dt=eps * eps,
                newton_tol=1e-8, gmres_tol=1e-10, gmres_restart=30)
    base.update(kw)
    return default_params(kind, **base)


def seeded_ic(nverts: int, seed: int, m: float, kind="ref") -> np.ndarray:
    lib = load(kind)
    u = np.empty(nverts)
    lib.oko_seeded_ic(nverts, seed, m, _p(u))
    return u


def mesh(dim: int, n: int, kind="ref"):
    lib = load(kind)
    s = n + 1
    nv = s ** dim
    nc = 2 * n * n if dim == 2 else 6 * n ** 3
    v = np.empty(nv * dim)
    c = np.empty(nc * (dim + 1), dtype=np.int32)
    _check(lib, lib.oko_mesh(dim, n, _p(v), c.ctypes.data_as(_ip)))
    return v.reshape(nv, dim), c.reshape(nc, dim + 1)


@dataclass
class NewtonStats:
    newton_iters: int
    gmres_iters: list
    residual_norm: float
    seconds: float
    converged: bool


class Oracle:
    """One reference context: mesh + operators + SchurContext."""

    def __init__(self, params: Params, kind: str = "ref"):
        self.kind = kind
        self.lib = load(kind)
        self.params = params
        st = C.c_int(0)
        self.h = self.lib.oko_create(C.byref(params), C.byref(st))
        if not self.h:
            raise OracleError(st.value, self.lib.oko_last_error().decode())
        self.n = self.lib.oko_num_vertices(self.h)

    def close(self):
        if self.h:
            self.lib.oko_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def levels(self):
        return self.lib.oko_levels(self.h)

    def level_size(self, level):
        return self.lib.oko_level_size(self.h, level)

    def scalars(self):
        out = np.empty(7)
        self.lib.oko_scalars(self.h, _p(out))
        keys = ["c", "sqrt_c", "a_coeff", "dt_theta", "lambda_lo", "lambda_hi", "eps_sqrt_c"]
        return dict(zip(keys, out.tolist()))

    def load_vector(self):
        b = np.empty(self.n)
        self.lib.oko_load_vector(self.h, _p(b))
        return b

    def level_dense(self, level):
        ns = self.level_size(level)
        a = np.empty(ns * ns)
        _check(self.lib, self.lib.oko_level_dense(self.h, level, _p(a)))
        return a.reshape(ns, ns)

    def set_linearization(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        _check(self.lib, self.lib.oko_set_linearization(self.h, _p(u)))

    def apply(self, kind, x, level=0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if kind == SHAT:
            out_n = self.level_size(level)
        elif kind == PROLONG:
            out_n = self.level_size(level)
        elif kind == RESTRICT:
            out_n = self.level_size(level + 1)
        elif kind in (BLOCK, JACOBIAN):
            out_n = 2 * self.n
        elif kind == COARSE_SOLVE:
            out_n = self.level_size(self.levels - 1)
        else:
            out_n = self.n
        y = np.empty(out_n)
        _check(self.lib, self.lib.oko_apply(self.h, kind, level, _p(x), _p(y)))
        return y

    def residual(self, un, wn, uo, wo):
        r1 = np.empty(self.n)
        r2 = np.empty(self.n)
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (un, wn, uo, wo)]
        _check(self.lib, self.lib.oko_residual(self.h, *[_p(a) for a in arrs], _p(r1), _p(r2)))
        return r1, r2

    def gmres(self, b, rtol, maxit, restart=0):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        it, conv, stag, nres = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        fres = C.c_double()
        cap = maxit + 2
        norms = np.empty(cap)
        _check(self.lib, self.lib.oko_gmres(self.h, _p(b), _p(x), rtol, maxit, restart,
                                            C.byref(it), C.byref(fres), C.byref(conv),
                                            C.byref(stag), _p(norms), cap, C.byref(nres)))
        return dict(x=x, iterations=it.value, final_residual=fres.value,
                    converged=bool(conv.value), stagnated=bool(stag.value),
                    residual_norms=norms[: min(nres.value, cap)].copy())

    def newton_solve(self, u_old, w_old):
        un = np.empty(self.n)
        wn = np.empty(self.n)
        ni, conv = C.c_int(), C.c_int()
        gi = np.zeros(max(self.params.newton_maxit, 1), dtype=np.int32)
        rn, secs = C.c_double(), C.c_double()
        uo = np.ascontiguousarray(u_old, dtype=np.float64)
        wo = np.ascontiguousarray(w_old, dtype=np.float64)
        _check(self.lib, self.lib.oko_newton_solve(self.h, _p(uo), _p(wo), _p(un), _p(wn),
                                                   C.byref(ni), gi.ctypes.data_as(_ip),
                                                   C.byref(rn), C.byref(secs), C.byref(conv)))
        stats = NewtonStats(ni.value, gi[: ni.value].tolist(), rn.value, secs.value,
                            bool(conv.value))
        return un, wn, stats

    def jacobi_spectrum(self):
        lo, hi = C.c_double(), C.c_double()
        _check(self.lib, self.lib.oko_jacobi_spectrum(self.h, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    # ---- diagnostics and initial state ----
    def total_mass(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = C.c_double()
        _check(self.lib, self.lib.oko_total_mass(self.h, _p(u), C.byref(out)))
        return out.value

    def double_well(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = C.c_double()
        _check(self.lib, self.lib.oko_double_well(self.h, _p(u), C.byref(out)))
        return out.value

    def energy(self, u):
        """-> (energy, cg_iters); cg_iters is -1 for the compiled reference (not exposed)."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        out, it = C.c_double(), C.c_int()
        _check(self.lib, self.lib.oko_energy(self.h, _p(u), C.byref(out), C.byref(it)))
        return out.value, it.value

    def initial_state(self):
        u, w = np.empty(self.n), np.empty(self.n)
        it = C.c_int()
        _check(self.lib, self.lib.oko_initial_state(self.h, _p(u), _p(w), C.byref(it)))
        return u, w, it.value


# ---- output formats of the compiled reference ----
# (through oracle/_ref/okref_io in a subprocess: numpy in this process breaks the
# reference's iostream/locale code)
REF_IO = os.path.join(HERE, "_ref", "okref_io")


def ref_format_g17(xs, workdir: str):
    import subprocess
    p = os.path.join(workdir, "fmt_in.bin")
    np.ascontiguousarray(xs, dtype=np.float64).tofile(p)
    out = subprocess.run([REF_IO, "fmt", p], capture_output=True, text=True, check=True)
    return out.stdout.splitlines()


def ref_write_vtk(dim: int, n: int, u, w, path: str, workdir: str) -> None:
    import subprocess
    p = os.path.join(workdir, "vtk_in.bin")
    np.concatenate([np.asarray(u, np.float64), np.asarray(w, np.float64)]).tofile(p)
    subprocess.run([REF_IO, "vtk", str(dim), str(n), p, path], capture_output=True, check=True)
