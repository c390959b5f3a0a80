"""C-ABI boundary checks that need no GPU: libokg.so loads, exports every
symbol include/okg.h declares, its host-side pieces (mesh arrays, seeded IC,
SolverConfig validation) match the reference, and on a machine without a GPU
context creation fails loudly instead of falling back to the CPU."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import pyoracle as po
from conftest import ROOT

import paper_1603_04570_b200 as okg
from paper_1603_04570_b200 import _lib

HEADER = os.path.join(ROOT, "include", "okg.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(okg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("okg_create", "okg_destroy", "okg_newton_step", "okg_apply", "okg_gmres", "okg_residual",
              "okg_linearize", "okg_mesh", "okg_set_state", "okg_get_state"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    out = subprocess.check_output(["nm", "-D", "--defined-only", _lib.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    for s in declared_symbols():
        getattr(_lib.lib, s)  # resolvable through ctypes


def test_library_is_sm100a():
    out = subprocess.check_output(["cuobjdump", "--list-elf", _lib.LIB_PATH], text=True)
    assert "sm_100a" in out


@pytest.mark.parametrize("dim,n", [(2, 1), (2, 5), (2, 16), (3, 1), (3, 4), (3, 9)])
def test_mesh_bit_exact(port_lib, dim, n):
    m = okg.build_mesh(dim, n)
    kind = "ref" if po.available("ref") else "port"
    v, c = po.mesh(dim, n, kind)
    assert np.array_equal(m.vertices, v)
    assert np.array_equal(m.cells, c)
    assert m.num_vertices() == (n + 1) ** dim
    assert m.num_cells() == (2 * n * n if dim == 2 else 6 * n ** 3)


def test_mesh_rejects_bad_arguments():
    with pytest.raises(okg.InvalidArgument):
        okg.build_mesh(4, 2)
    with pytest.raises(okg.InvalidArgument):
        okg.build_mesh(2, 0)


def test_seeded_ic_matches_oracle(port_lib):
    for seed, m in [(0, 0.0), (1, 0.1), (2, -0.4)]:
        a = okg.seeded_ic(5000, seed, m)
        assert np.array_equal(a, po.seeded_ic(5000, seed, m, "port"))
        assert np.all(np.abs(a - m) <= 0.01)


def test_default_config_matches_reference(port_lib):
    ref = po.default_params("port")
    cfg = okg.SolverConfig()
    for f in ("dim", "n", "eps", "sigma", "m", "theta", "dt", "newton_tol", "newton_maxit", "gmres_tol",
              "gmres_maxit", "gmres_restart", "cheby_iters", "richardson_steps", "mg_cycles", "mg_pre",
              "mg_post", "mg_omega", "min_coarse_size"):
        assert getattr(cfg, f) == getattr(ref, f), f
    p = _lib.Params()
    assert _lib.lib.okg_default_params(C.byref(p)) == 0
    assert p.gmres_maxit == 200 and p.use_graphs == 1


@pytest.mark.parametrize("field,value", [("eps", 0.0), ("sigma", -1.0), ("m", 1.0), ("theta", 0.0),
                                         ("theta", 1.5), ("dt", 0.0), ("n", 0), ("newton_tol", 0.0),
                                         ("newton_maxit", 0), ("gmres_tol", 0.0), ("gmres_maxit", 0),
                                         ("gmres_restart", -1), ("cheby_iters", 0), ("richardson_steps", 0),
                                         ("mg_cycles", 0), ("mg_omega", 2.0), ("min_coarse_size", 0),
                                         ("cheby_precond", "sor"), ("max_dofs", 0)])
def test_validate_rejects(field, value):
    # SolverConfig::validate, params.hpp:68-116
    cfg = okg.SolverConfig()
    setattr(cfg, field, value)
    with pytest.raises(okg.ConfigError):
        cfg.validate()


def test_validate_vertex_cap():
    okg.SolverConfig().validate()
    with pytest.raises(okg.ConfigError, match="max_dofs"):
        okg.SolverConfig(dim=3, n=128).validate()
    okg.SolverConfig(dim=3, n=128, max_dofs=3_000_000).validate()


def test_compute_c():
    assert abs(okg.compute_c(0.0004, 0.5, 100.0) - 0.00019607843137254902) <= 1e-15 * 2e-4
    assert okg.compute_c(1.0, 0.5, 0.0) == 0.5
    for bad in [(0.0, 0.5, 100.0), (1e-4, 0.0, 100.0), (1e-4, 1.5, 100.0), (1e-4, 0.5, -1.0)]:
        with pytest.raises(okg.InvalidArgument):
            okg.compute_c(*bad)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    with pytest.raises(okg.CudaError):
        okg.SchurContext(okg.SolverConfig(dim=2, n=8))
