"""Field sketches for parity at BASELINE sizes -- TEST INFRASTRUCTURE ONLY.

A full-size field (up to 4.2 M doubles at 2D 2048^2 / 3D 128^3) is too large to
commit per timestep, so the reference fixtures (tests/golden/make_baseline_fixtures.py)
store, per timestep, the norm of u and w and NPROJ Rademacher projections
p_k = sum_g s_k(g) x(g), s_k(g) in {-1, +1}.  For an error field e = x - x_ref the
projections give an unbiased estimate of its squared norm:

    E[(s_k . e)^2] = ||e||^2,   so   ||e||^2 ~= mean_k (p_k(x) - p_k(x_ref))^2

(64 projections: the estimate is within a factor ~1.5 of ||e|| with overwhelming
probability, ample for a 1e-8 bound).  The signs are counter-based (one splitmix64
hash per global vertex id gives the 64 sign bits of that vertex), so any host
regenerates them from the vertex count alone.
"""
from __future__ import annotations

import numpy as np

NPROJ = 64
SKETCH_KEY = np.uint64(0x5EED5EED0C0FFEE1)
_CHUNK = 1 << 18


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def _signs(g0: int, g1: int) -> np.ndarray:
    """(g1-g0, 64) float64 matrix of +-1 for global vertex ids [g0, g1)."""
    g = np.arange(g0, g1, dtype=np.uint64)
    h = _splitmix64(g ^ SKETCH_KEY)
    bits = np.unpackbits(h.view(np.uint8).reshape(-1, 8), axis=1)  # (n, 64)
    return 1.0 - 2.0 * bits.astype(np.float64)


def project(*fields: np.ndarray) -> np.ndarray:
    """-> (len(fields), NPROJ) projections of each field (all of one length N)."""
    X = np.stack([np.ascontiguousarray(f, dtype=np.float64) for f in fields], axis=1)
    n = X.shape[0]
    out = np.zeros((NPROJ, X.shape[1]))
    for g0 in range(0, n, _CHUNK):
        g1 = min(n, g0 + _CHUNK)
        out += _signs(g0, g1).T @ X[g0:g1]
    return out.T.copy()


def sketch(u: np.ndarray, w: np.ndarray) -> dict:
    p = project(u, w)
    return {"norm_u": float(np.linalg.norm(u)), "norm_w": float(np.linalg.norm(w)),
            "proj_u": p[0], "proj_w": p[1]}


def est_relerr(proj: np.ndarray, proj_ref: np.ndarray, norm_ref: float) -> float:
    """Estimated ||x - x_ref|| / ||x_ref|| from the two projection vectors."""
    d = np.asarray(proj) - np.asarray(proj_ref)
    e = float(np.sqrt(np.mean(d * d)))
    return e / (norm_ref if norm_ref > 0 else 1.0)
