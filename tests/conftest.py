import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: larger sizes")


def golden_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "d*.npz")))


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def golden_params(g, kind="port"):
    import pyoracle as po
    return po.baseline_params(int(g["dim"]), int(g["n"]), eps=float(g["eps"]), m=float(g["m"]),
                              kind=kind, min_coarse_size=int(g["min_coarse"]), cheby_ssor=int(g.get("ssor", 0)))


def golden_config(g):
    import paper_1603_04570_b200 as okg
    return okg.SolverConfig(dim=int(g["dim"]), n=int(g["n"]), eps=float(g["eps"]), m=float(g["m"]),
                            dt=float(g["eps"]) ** 2, sigma=100.0, theta=0.5, newton_tol=1e-8,
                            gmres_tol=1e-10, gmres_restart=30, min_coarse_size=int(g["min_coarse"]),
                            cheby_precond="ssor" if int(g.get("ssor", 0)) else "jacobi")


def relerr(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="session")
def port_lib():
    import pyoracle as po
    if not po.available("port"):
        import subprocess
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "port"])
    return po.load("port")
