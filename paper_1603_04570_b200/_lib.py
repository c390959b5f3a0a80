"""ctypes binding of include/okg.h (libokg.so, the sm_100a Newton linear solver).

The product path: no CPU fallback.  If ``libokg.so`` is missing this module
raises at import time; if no CUDA device is present, context creation fails
with ``CudaError`` (status OKG_ECUDA) -- nothing silently runs on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OKG_LIB") or os.path.join(HERE, "libokg.so")  # OKG_LIB: A/B builds (tools)

OKG_OK = 0
OKG_EINVAL = -1
OKG_ENUMERICAL = -2
OKG_ECONFIG = -3
OKG_EINCONSISTENT = -4
OKG_ECOARSEN = -5
OKG_ECUDA = -6
OKG_ENOMEM = -7
OKG_EOTHER = -9

OP_M, OP_K, OP_A, OP_SHAT, OP_PROLONG, OP_RESTRICT, OP_VCYCLE, OP_SHAT_INV = range(8)
OP_CHEB_M, OP_CHEB_A, OP_ME, OP_C, OP_SCHUR, OP_SCHUR_TILDE_INV = range(8, 14)
OP_S_INV_APPROX, OP_BLOCK, OP_JACOBIAN, OP_NONLINEAR, OP_COARSE_SOLVE, OP_SSOR_M = range(14, 20)

OKG_MAX_NEWTON = 64

KT_NAMES = ["smooth", "resid", "pre2", "post_acc", "cheb", "jacobian", "restrict", "prolong"]
KT_COLD, KT_NO_PDL = 1, 2


class Params(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("n", C.c_int32),
        ("eps", C.c_double), ("sigma", C.c_double), ("m", C.c_double),
        ("theta", C.c_double), ("dt", C.c_double),
        ("newton_tol", C.c_double), ("newton_maxit", C.c_int32),
        ("gmres_tol", C.c_double), ("gmres_maxit", C.c_int32), ("gmres_restart", C.c_int32),
        ("cheby_iters", C.c_int32), ("richardson_steps", C.c_int32),
        ("mg_cycles", C.c_int32), ("mg_pre", C.c_int32), ("mg_post", C.c_int32),
        ("mg_omega", C.c_double), ("min_coarse_size", C.c_int32),
        ("shat_perturb", C.c_double), ("max_dofs", C.c_int64),
        ("device", C.c_int32), ("use_graphs", C.c_int32), ("tiled_min_n", C.c_int32),
        ("tail_max_vertices", C.c_int32), ("disable_pdl", C.c_int32),
        ("mg_fuse", C.c_int32), ("nslabs", C.c_int32), ("slab_devices", C.c_int32),
        ("tail_cluster", C.c_int32),
        ("cheby_ssor", C.c_int32),
        ("coarse_split", C.c_int32),
        ("mg_collapse", C.c_int32),
        ("rep_max_vertices", C.c_int64),
    ]


class StepStats(C.Structure):
    _fields_ = [
        ("step", C.c_int32), ("t", C.c_double), ("newton_iters", C.c_int32),
        ("gmres_iters", C.c_int32 * OKG_MAX_NEWTON), ("residual_norm", C.c_double),
        ("seconds", C.c_double), ("converged", C.c_int32), ("kernel_launches", C.c_int64),
        ("mass", C.c_double), ("energy", C.c_double),
    ]


class KrylovStats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("converged", C.c_int32), ("stagnated", C.c_int32),
        ("final_residual", C.c_double), ("n_residual_norms", C.c_int32),
        ("residual_norms", C.c_double * 512),
    ]


class Info(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("n", C.c_int32), ("num_vertices", C.c_int64),
        ("levels", C.c_int32), ("level_size", C.c_int64 * 32), ("level_n", C.c_int32 * 32),
        ("c", C.c_double), ("sqrt_c", C.c_double), ("a_coeff", C.c_double),
        ("dt_theta", C.c_double), ("lambda_lo", C.c_double), ("lambda_hi", C.c_double),
        ("eps_sqrt_c", C.c_double), ("device_bytes", C.c_int64), ("graph_nodes", C.c_int32),
        ("tail_start", C.c_int32), ("tiled_mask", C.c_int32),
        ("nslabs", C.c_int32), ("rep_level", C.c_int32),
        ("slab_ilo", C.c_int32 * 16), ("slab_ihi", C.c_int32 * 16), ("tail_cluster", C.c_int32),
        ("coarse_rows", C.c_int32), ("collapse_level", C.c_int32),
    ]


# --- the reference's exception types (errors.hpp:9-28), raised by the host mirror ---
class OkgError(RuntimeError):
    status = OKG_EOTHER


class InvalidArgument(OkgError, ValueError):   # std::invalid_argument
    status = OKG_EINVAL


class NumericalError(OkgError):               # okflow::NumericalError
    status = OKG_ENUMERICAL


class ConfigError(OkgError):                  # okflow::ConfigError
    status = OKG_ECONFIG


class InconsistentState(OkgError):            # okflow::InconsistentState
    status = OKG_EINCONSISTENT


class CannotCoarsen(OkgError):                # okflow::CannotCoarsen
    status = OKG_ECOARSEN


class CudaError(OkgError):
    status = OKG_ECUDA


class DeviceOutOfMemory(OkgError):
    status = OKG_ENOMEM


_ERR = {c.status: c for c in (InvalidArgument, NumericalError, ConfigError, InconsistentState,
                              CannotCoarsen, CudaError, DeviceOutOfMemory)}

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_1603_04570_b200/csrc)")

lib = C.CDLL(LIB_PATH)

_SIGS = {
    "okg_default_params": (C.c_int, [C.POINTER(Params)]),
    "okg_validate_params": (C.c_int, [C.POINTER(Params)]),
    "okg_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
    "okg_create": (C.c_int, [C.POINTER(Params), C.POINTER(_vp)]),
    "okg_destroy": (None, [_vp]),
    "okg_get_info": (C.c_int, [_vp, C.POINTER(Info)]),
    "okg_mesh": (C.c_int, [C.c_int32, C.c_int32, _dp, C.POINTER(C.c_int32)]),
    "okg_seeded_ic": (C.c_int, [C.c_int64, C.c_uint64, C.c_double, _dp]),
    "okg_set_state": (C.c_int, [_vp, _dp, _dp, C.c_double, C.c_int32]),
    "okg_get_state": (C.c_int, [_vp, _dp, _dp, C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
    "okg_newton_step": (C.c_int, [_vp, C.POINTER(StepStats)]),
    "okg_newton_step_host": (C.c_int, [_vp, _dp, _dp, _dp, _dp, C.POINTER(StepStats)]),
    "okg_linearize": (C.c_int, [_vp, _vp]),
    "okg_clear_linearization": (C.c_int, [_vp]),
    "okg_apply": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp]),
    "okg_residual": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "okg_gmres": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int32, C.c_int32, C.POINTER(KrylovStats)]),
    "okg_jacobi_spectrum": (C.c_int, [_vp, _dp, _dp]),
    "okg_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "okg_slab_stream": (C.c_int, [_vp, C.c_int32, C.POINTER(_vp)]),
    "okg_nccl_unique_id": (C.c_int, [_vp, C.c_size_t]),
    "okg_total_mass": (C.c_int, [_vp, _dp, _dp]),
    "okg_double_well": (C.c_int, [_vp, _dp, _dp]),
    "okg_energy": (C.c_int, [_vp, _dp, _dp, C.POINTER(C.c_int32)]),
    "okg_initial_state": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "okg_advance": (C.c_int, [_vp, C.c_int32, C.POINTER(StepStats)]),
    "okg_create_rank": (C.c_int, [C.POINTER(Params), C.c_int32, C.c_int32, _vp, C.POINTER(_vp)]),
    "okg_slab_partition": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32)]),
    "okg_linearize_host": (C.c_int, [_vp, _dp]),
    "okg_apply_host": (C.c_int, [_vp, C.c_int32, C.c_int32, _dp, _dp]),
    "okg_residual_host": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, _dp]),
    "okg_gmres_host": (C.c_int, [_vp, _dp, _dp, C.c_double, C.c_int32, C.c_int32, C.POINTER(KrylovStats)]),
    "okg_apply_host_n": (C.c_int, [_vp, C.c_int32, C.c_int32, _dp, C.c_int64, _dp, C.c_int64]),
    "okg_linearize_host_n": (C.c_int, [_vp, _dp, C.c_int64]),
    "okg_residual_host_n": (C.c_int, [_vp, _dp, _dp, _dp, _dp, C.c_int64, _dp, _dp]),
    "okg_gmres_host_n": (C.c_int, [_vp, _dp, _dp, C.c_int64, C.c_double, C.c_int32, C.c_int32,
                                   C.POINTER(KrylovStats)]),
    "okg_kernel_timing": (C.c_int, [_vp, C.c_int32, C.c_int32, _dp, _dp]),
    "okg_kernel_timing_ex": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, _dp, _dp]),
    "okg_device_alloc": (C.c_int, [C.c_int32, C.c_size_t, C.POINTER(_vp)]),
    "okg_device_free": (C.c_int, [_vp]),
    "okg_memcpy_h2d": (C.c_int, [_vp, _vp, C.c_size_t]),
    "okg_memcpy_d2h": (C.c_int, [_vp, _vp, C.c_size_t]),
    "okg_device_synchronize": (C.c_int, []),
    "okg_kernel_launch_count": (C.c_int64, []),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def last_error() -> str:
    buf = C.create_string_buffer(2048)
    lib.okg_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(status: int):
    if status != OKG_OK:
        raise _ERR.get(status, OkgError)(last_error())
