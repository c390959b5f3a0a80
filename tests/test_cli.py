"""INI front end, study drivers and command line.

parse_config of the Python (paper_1603_04570_b200.cli) and C++ (okg/okflow_cli.hpp)
mirrors against the reference's own config.hpp (oracle/_ref/okref_io cfg) on
valid files and on every error path: same values, same ConfigError messages.
The GPU tests run the command lines end to end."""
import os
import subprocess
import sys

import pytest

import pyoracle as po
from conftest import ROOT

import paper_1603_04570_b200 as okg
from paper_1603_04570_b200 import cli
from paper_1603_04570_b200.io import format_g17

CPP = os.path.join(ROOT, "tests", "cpp", "test_okflow_io")
CLI_BIN = os.path.join(ROOT, "paper_1603_04570_b200", "okflow_b200")
need_ref = pytest.mark.skipif(not os.path.exists(po.REF_IO), reason="oracle/_ref not built")

REQ = "[problem]\neps = 0.02\nsigma = 100\nm = 0.1\ntheta = 0.5\n[mesh]\ndim = 2\nn = 16\n[solver]\ndt = 4e-4\nn_steps = 2\n"

CASES = {
    "minimal": REQ,
    "full": ("# a comment line\n; another\n[problem]\n  eps = 0.01   # inline comment\nsigma=50\nm = -0.25 ; c\n"
             "theta = 1\neps_list = 0.04, 0.02 ,, 0.01\n\n[mesh]\ndim = 3\nn = 8\nmesh_study_n = 4, 8\n"
             "max_dofs = 5000\n[solver]\ndt = 0x1p-12\nn_steps = 0\nnewton_tol = 1e-9\nnewton_maxit = 7\n"
             "gmres_tol = +1e-10\ngmres_maxit = 50\ngmres_restart = 30\ncheby_iters = 8\ncheby_precond = ssor\n"
             "richardson_steps = 3\nmg_cycles = 4\nmg_pre = 1\nmg_post = 3\nmg_omega = 0.7\n"
             "min_coarse_size = 64\nthreads = 4\n[output]\ndirectory = out#1 ; kept glued marker\n"
             "snapshot_every = 5\n"),
    "crlf": REQ.replace("\n", "\r\n"),
    "spaces_in_section": REQ.replace("[mesh]", "[ mesh ]"),
    "unknown_section": REQ + "[extra]\nx = 1\n",
    "unknown_key": REQ + "[solver]\ntolerance = 1\n",
    "malformed_header": REQ + "[output\n",
    "no_equals": REQ + "[solver]\nmg_cycles 4\n",
    "outside_section": "eps = 0.02\n" + REQ,
    "empty_key": REQ + "[solver]\n = 3\n",
    "missing_required": REQ.replace("theta = 0.5\n", ""),
    "bad_double": REQ.replace("eps = 0.02", "eps = 0.02x"),
    "bad_int": REQ.replace("n = 16", "n = 16.5"),
    "empty_value": REQ.replace("n = 16", "n ="),
    "empty_list": REQ + "[problem]\neps_list = , ,\n",
    "bad_list_item": REQ + "[mesh]\nmesh_study_n = 8, x\n",
    "invalid_theta": REQ.replace("theta = 0.5", "theta = 1.5"),
    "invalid_dim": REQ.replace("dim = 2", "dim = 4"),
    "invalid_precond": REQ + "[solver]\ncheby_precond = ilu\n",
    "too_big": REQ + "[mesh]\nmax_dofs = 100\n",
    "bad_study_n": REQ + "[mesh]\nmesh_study_n = 8, 0\n",
    "negative_snapshot": REQ + "[output]\nsnapshot_every = -1\n",
    "duplicate_key_last_wins": REQ + "[mesh]\nn = 32\n",
}


def py_dump(path):
    try:
        c = cli.parse_config(path).config
    except okg.ConfigError as e:
        return f"ERR -3: {e}\n"
    d = lambda k, v: f"{k}={format_g17(v)}\n"  # noqa: E731
    i = lambda k, v: f"{k}={v}\n"  # noqa: E731
    return (d("eps", c.eps) + d("sigma", c.sigma) + d("m", c.m) + d("theta", c.theta) + d("dt", c.dt)
            + i("n_steps", c.n_steps) + i("dim", c.dim) + i("n", c.n) + d("newton_tol", c.newton_tol)
            + i("newton_maxit", c.newton_maxit) + d("gmres_tol", c.gmres_tol) + i("gmres_maxit", c.gmres_maxit)
            + i("gmres_restart", c.gmres_restart) + i("cheby_iters", c.cheby_iters)
            + f"cheby_precond={c.cheby_precond}\n" + i("richardson_steps", c.richardson_steps)
            + i("mg_cycles", c.mg_cycles) + i("mg_pre", c.mg_pre) + i("mg_post", c.mg_post)
            + d("mg_omega", c.mg_omega) + i("min_coarse_size", c.min_coarse_size) + i("threads", c.threads)
            + i("max_dofs", c.max_dofs) + f"output_dir={c.output_dir}\n" + i("snapshot_every", c.snapshot_every)
            + "mesh_study_n=" + ",".join(str(x) for x in c.mesh_study_n) + "\n"
            + "eps_list=" + ",".join(format_g17(x) for x in c.eps_list) + "\n")


@pytest.fixture
def ini(tmp_path):
    def make(name):
        p = tmp_path / f"{name}.ini"
        p.write_bytes(CASES[name].encode())
        return str(p)
    return make


@need_ref
@pytest.mark.parametrize("name", sorted(CASES))
def test_parse_config_matches_reference(ini, name):
    path = ini(name)
    ref = subprocess.run([po.REF_IO, "cfg", path], capture_output=True, text=True, check=True).stdout
    assert py_dump(path) == ref
    if os.path.exists(CPP):
        cpp = subprocess.run([CPP, "cfg", path], capture_output=True, text=True, check=True).stdout
        assert cpp == ref


def test_parse_config_missing_file(tmp_path):
    with pytest.raises(okg.ConfigError, match="config: cannot open file"):
        cli.parse_config(str(tmp_path / "nope.ini"))


def test_cli_config_error_exit_code(ini, capsys):
    assert cli.main(["run", "--config", ini("invalid_theta")]) == 2
    assert "config error: config: theta must lie in (0, 1]" in capsys.readouterr().err
    if os.path.exists(CLI_BIN):
        out = subprocess.run([CLI_BIN, "run", "--config", ini("unknown_key")], capture_output=True, text=True)
        assert out.returncode == 2 and "config error: config: unknown key 'tolerance'" in out.stderr


def test_cli_verify_is_reference_only(ini):
    assert cli.main(["verify", "--config", ini("minimal")]) == 1


@pytest.mark.gpu
def test_cli_run_python_and_cpp(tmp_path, ini):
    path = ini("minimal")
    for tag, cmd in (("py", [sys.executable, "-m", "paper_1603_04570_b200"]), ("cpp", [CLI_BIN])):
        if tag == "cpp" and not os.path.exists(CLI_BIN):
            continue
        d = tmp_path / tag
        out = subprocess.run(cmd + ["run", "--config", path, "--output", str(d)], capture_output=True, text=True,
                             cwd=ROOT)
        assert out.returncode == 0, out.stderr
        assert out.stdout.startswith("run: 2 steps, 2D n=16, avg GMRES per Newton = ")
        rows = (d / "stats.csv").read_text().splitlines()
        assert len(rows) == 3 and rows[0].startswith("step,newton_iters")
        assert (d / "state_0.vtk").exists()


@pytest.mark.gpu
def test_mesh_and_eps_study(tmp_path):
    p = tmp_path / "s.ini"
    p.write_text(REQ + "[problem]\neps_list = 0.25, 0.125\n[mesh]\nmesh_study_n = 8, 16\n")
    for kind, csv, header, nrows in (("mesh-study", "mesh_study.csv", "n,dofs,avg_gmres_per_newton", 2),
                                     ("eps-study", "eps_study.csv", "eps,dx,dt,avg_gmres_per_newton", 2)):
        d = tmp_path / kind
        assert cli.main([kind, "--config", str(p), "--output", str(d)]) == 0
        rows = (d / csv).read_text().splitlines()
        assert rows[0] == header and len(rows) == nrows + 1
    rows = (tmp_path / "eps-study" / "eps_study.csv").read_text().splitlines()
    assert rows[1].startswith("0.25,0.125,0.0625,") and rows[2].startswith("0.125,0.0625,0.015625,")
    # the eps-study refuses meshes above max_dofs up front (exit 2)
    q = tmp_path / "big.ini"
    q.write_text(REQ + "[problem]\neps_list = 0.001\n")
    assert cli.main(["eps-study", "--config", str(q), "--output", str(tmp_path / "big")]) == 2
