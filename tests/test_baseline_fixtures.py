"""CPU checks of the BASELINE-size fixtures (tests/golden/baseline) and of the
field-sketch estimator the GPU test (test_gpu_baseline_full.py) relies on."""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN
from sketch import NPROJ, est_relerr, project

# first-step counts the reference took in SURVEY.md section 6 (measured there independently)
SURVEY_FIRST = {"c2_n128": 12, "c2_n256": 11, "c2_n512": 10, "c2_n1024": 9, "c2_n2048": 9,
                "c3_e040": 9, "c3_e020": 9, "c3_e010": 10, "c3_e005": 11, "c4_3d128": 12}
PATHS = sorted(glob.glob(os.path.join(GOLDEN, "baseline", "*.npz")))


def load(p):
    with np.load(p) as z:
        return {k: z[k] for k in z.files}


def test_estimator_tracks_true_error():
    rng = np.random.default_rng(7)
    x = rng.standard_normal(100_003)
    for scale in (1e-14, 1e-10, 1e-6):
        e = scale * rng.standard_normal(x.size)
        px, py = project(x, x + e)
        est = est_relerr(py, px, np.linalg.norm(x))
        true = np.linalg.norm(e) / np.linalg.norm(x)
        assert 0.5 * true <= est <= 2.0 * true, (scale, est, true)
    assert project(x).shape == (1, NPROJ)


def test_signs_are_counter_based():
    """chunking does not change the projections (signs depend on the vertex id only)"""
    import sketch
    x = np.random.default_rng(3).standard_normal(300_001)
    a = project(x)
    old = sketch._CHUNK
    try:
        sketch._CHUNK = 1 << 12
        b = project(x)
    finally:
        sketch._CHUNK = old
    assert np.allclose(a, b, rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("path", PATHS, ids=[os.path.basename(p)[:-4] for p in PATHS])
def test_fixture_consistent(path):
    f = load(path)
    name = os.path.basename(path)[:-4]
    steps = int(f["steps"])
    assert f["newton_iters"].shape == (steps,) and f["proj_u"].shape == (steps, NPROJ)
    assert all(f["converged"]) and all(int(k) == 1 for k in f["newton_iters"])
    assert int(f["gmres_iters"][0][0]) == SURVEY_FIRST[name]
    for k in range(steps):
        if f"u{k + 1}" in f:
            p = project(f[f"u{k + 1}"], f[f"w{k + 1}"])
            assert np.allclose(p[0], f["proj_u"][k], rtol=1e-12, atol=1e-12)
            assert np.allclose(p[1], f["proj_w"][k], rtol=1e-12, atol=1e-12)
            assert np.isclose(np.linalg.norm(f[f"u{k + 1}"]), f["norm_u"][k], rtol=1e-14)


def test_port_matches_fixture_every_step(port_lib):
    """the plain-C oracle (bit-exact to the reference) replays configs[1] 128^2 x 5 steps"""
    import pyoracle as po
    f = load(os.path.join(GOLDEN, "baseline", "c2_n128.npz"))
    o = po.Oracle(po.baseline_params(2, 128, kind="port"), "port")
    u = po.seeded_ic(o.n, 0, 0.0, "port")
    w = np.zeros(o.n)
    for k in range(int(f["steps"])):
        u, w, st = o.newton_solve(u, w)
        assert st.gmres_iters == [int(x) for x in f["gmres_iters"][k] if x >= 0]
        assert np.array_equal(u, f[f"u{k + 1}"]) and np.array_equal(w, f[f"w{k + 1}"])
