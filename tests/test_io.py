"""Output formats: format_g17, the VTK snapshot and stats.csv rows
of the Python (paper_1603_04570_b200.io) and C++ (include/okg/okflow_io.hpp)
mirrors against the reference's own vtk.hpp (oracle/_ref/okref_io) and its
golden-bytes test (test_cli.cpp:138-163).  CPU only, except the cmd_run tests."""
import os
import subprocess

import numpy as np
import pytest

import pyoracle as po
from conftest import ROOT

import paper_1603_04570_b200 as okg
from paper_1603_04570_b200 import io

CPP = os.path.join(ROOT, "tests", "cpp", "test_okflow_io")
need_ref = pytest.mark.skipif(not os.path.exists(po.REF_IO), reason="oracle/_ref not built")
need_cpp = pytest.mark.skipif(not os.path.exists(CPP), reason="tests/cpp/test_okflow_io not built")

VALUES = np.concatenate([np.random.default_rng(11).uniform(-1e3, 1e3, 500),
                         np.random.default_rng(12).standard_normal(500) * 1e-7,
                         [0.0, -0.0, 0.5, 1.0, -2.5, 1e-300, 1e300, 5e-324, 1 / 3, 2 / 3, 0.1, 1e16, 123456789.0]])


def test_format_g17_kats():
    # test_cli.cpp:124-136
    assert io.format_g17(0.0) == "0" and io.format_g17(0.5) == "0.5" and io.format_g17(1.0) == "1"
    for x in VALUES:
        assert float(io.format_g17(x)) == x


@need_ref
def test_format_g17_matches_reference(tmp_path):
    assert [io.format_g17(x) for x in VALUES] == po.ref_format_g17(VALUES, str(tmp_path))


@need_ref
@need_cpp
def test_cpp_format_g17_matches_reference(tmp_path):
    p = tmp_path / "v.bin"
    VALUES.astype(np.float64).tofile(p)
    out = subprocess.run([CPP, "fmt", str(p)], capture_output=True, text=True, check=True).stdout.splitlines()
    assert out == po.ref_format_g17(VALUES, str(tmp_path))


def test_vtk_golden_bytes(tmp_path):
    """test_cli.cpp:138-163: a 2x2 mesh of zeros."""
    p = tmp_path / "state_0.vtk"
    io.write_vtk(2, 2, np.zeros(9), np.zeros(9), str(p))
    zeros = "0\n" * 9
    golden = ("# vtk DataFile Version 3.0\nokflow state\nASCII\nDATASET STRUCTURED_POINTS\n"
              "DIMENSIONS 3 3 1\nORIGIN 0 0 0\nSPACING 0.5 0.5 0.5\nPOINT_DATA 9\n"
              "SCALARS u double 1\nLOOKUP_TABLE default\n" + zeros +
              "SCALARS w double 1\nLOOKUP_TABLE default\n" + zeros)
    assert p.read_bytes() == golden.encode()


@pytest.mark.parametrize("dim,n", [(2, 1), (2, 4), (2, 7), (3, 2), (3, 5)])
def test_vtk_round_trip_native_order(tmp_path, dim, n):
    """test_cli.cpp:165-: values round-trip in the format's native point order (x fastest)."""
    s = n + 1
    mesh = okg.build_mesh(dim, n)
    u = mesh.vertices[:, 0] + 10.0 * mesh.vertices[:, 1] + (100.0 * mesh.vertices[:, 2] if dim == 3 else 0.0)
    w = np.random.default_rng(5).uniform(-1, 1, mesh.num_vertices())
    p = tmp_path / "f.vtk"
    io.write_vtk(dim, n, u, w, str(p))
    lines = p.read_text().splitlines()
    i0 = lines.index("SCALARS u double 1") + 2
    uu = np.array([float(x) for x in lines[i0:i0 + s ** dim]])
    # native order: point (i, j, k) at (k * s + j) * s + i
    for v in range(mesh.num_vertices()):
        i, j, k = mesh.grid_coords(v)
        assert uu[(k * s + j) * s + i] == u[v]
    wi = lines.index("SCALARS w double 1") + 2
    ww = np.array([float(x) for x in lines[wi:wi + s ** dim]])
    assert np.array_equal(np.sort(ww), np.sort(w))


@need_ref
@pytest.mark.parametrize("dim,n", [(2, 3), (2, 16), (3, 4), (3, 7)])
def test_vtk_bytes_match_reference(tmp_path, dim, n):
    N = (n + 1) ** dim
    rng = np.random.default_rng(dim * 100 + n)
    u = rng.standard_normal(N) * 10.0 ** rng.integers(-8, 8, N)
    w = rng.uniform(-1, 1, N)
    ref, ours = tmp_path / "ref.vtk", tmp_path / "ours.vtk"
    po.ref_write_vtk(dim, n, u, w, str(ref), str(tmp_path))
    io.write_vtk(dim, n, u, w, str(ours))
    assert ours.read_bytes() == ref.read_bytes()
    if os.path.exists(CPP):
        cpp = tmp_path / "cpp.vtk"
        inp = tmp_path / "in.bin"
        np.concatenate([u, w]).tofile(inp)
        subprocess.run([CPP, "vtk", str(dim), str(n), str(inp), str(cpp)], check=True)
        assert cpp.read_bytes() == ref.read_bytes()


def test_vtk_size_mismatch(tmp_path):
    with pytest.raises(okg.InconsistentState):
        io.write_vtk(2, 2, np.zeros(8), np.zeros(9), str(tmp_path / "x.vtk"))


def test_stats_row_format():
    """driver.hpp:87-101: step,newton_iters,total_gmres,avg_gmres,residual,mass,energy,seconds"""
    st = okg.IterationStats(step=3, newton_iters=2, gmres_iters=[13, 14], residual_norm=1.25e-9, mass=0.1,
                            energy=0.2450384537810161, seconds=0.5)
    assert io.stats_row(st) == "3,2,27,13.5,1.25e-09,0.10000000000000001,0.2450384537810161,0.5\n"
    assert io.STATS_HEADER == "step,newton_iters,total_gmres,avg_gmres,residual,mass,energy,seconds\n"


def _check_run_dir(d, dim, n, steps, every):
    rows = (d / "stats.csv").read_text().splitlines()
    assert rows[0] == io.STATS_HEADER.strip() and len(rows) == steps + 1
    for k, r in enumerate(rows[1:], start=1):
        f = r.split(",")
        assert int(f[0]) == k and int(f[1]) >= 1 and int(f[2]) >= int(f[1])
        assert abs(float(f[5]) - 0.1) <= 1e-12  # mass conserved
    snaps = sorted(p.name for p in d.glob("state_*.vtk"))
    want = sorted({"state_0.vtk"} | {f"state_{k}.vtk" for k in range(every, steps + 1, every)})
    assert snaps == want
    return rows


@pytest.mark.gpu
def test_cmd_run_python(tmp_path):
    cfg = okg.SolverConfig(dim=2, n=16, m=0.1, dt=4e-4, n_steps=3, gmres_tol=1e-10, gmres_restart=30)
    assert io.cmd_run(cfg, str(tmp_path), snapshot_every=2) == 0
    _check_run_dir(tmp_path, 2, 16, 3, 2)
    # the initial snapshot holds initial_state's u0
    o = po.Oracle(po.baseline_params(2, 16, m=0.1, kind="port", dt=4e-4), "port")
    u0, _, _ = o.initial_state()
    lines = (tmp_path / "state_0.vtk").read_text().splitlines()
    i0 = lines.index("SCALARS u double 1") + 2
    uu = np.array([float(x) for x in lines[i0:i0 + 17 * 17]]).reshape(17, 17).T.reshape(-1)
    assert np.max(np.abs(uu - u0)) <= 1e-16


@pytest.mark.gpu
@need_cpp
def test_cmd_run_cpp(tmp_path):
    out = subprocess.run([CPP, "run", "3", "8", "2", "1", str(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("run: 2 steps, 3D n=8, avg GMRES per Newton = ")
    _check_run_dir(tmp_path, 3, 8, 2, 1)
