"""Localisation accuracy of PAPER.md §4: the DOA mappings f_1, f_2, f_3 and the energy-weighted RMSE
of eq. `results_rmse`.  Float64, plain numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): tools/fig2a_rmse.py and tests/ call it to turn DOA indices and
scores (from the oracle or from the CUDA path) into the paper's accuracy figure; the product path never imports it.
"""
from __future__ import annotations

import numpy as np


def g_elevation(s: np.ndarray) -> np.ndarray:
    """g(s) = atan2{ s|_z, sqrt(s|_x^2 + s|_y^2) }.  s (..., 3) -> (...)."""
    s = np.asarray(s, dtype=np.float64)
    return np.arctan2(s[..., 2], np.sqrt(s[..., 0] ** 2 + s[..., 1] ** 2))


def f1(s: np.ndarray) -> np.ndarray:
    """1-D linear array: the 3-D position is mapped to the 180 degree arc, f_1(s) = [cos g, 0, sin g]."""
    g = g_elevation(s)
    return np.stack([np.cos(g), np.zeros_like(g), np.sin(g)], axis=-1)


def f2(s: np.ndarray) -> np.ndarray:
    """2-D planar array: every point is mapped to the positive hemisphere, f_2(s) = [s_x, s_y, |s_z|]."""
    s = np.asarray(s, dtype=np.float64)
    return np.stack([s[..., 0], s[..., 1], np.abs(s[..., 2])], axis=-1)


def f3(s: np.ndarray) -> np.ndarray:
    """3-D array: identity."""
    return np.asarray(s, dtype=np.float64).copy()


MAPS = {1: f1, 2: f2, 3: f3}


def rmse(alpha: int, s_est: np.ndarray, Y: np.ndarray, s0: np.ndarray) -> float:
    """Eq. results_rmse: RMSE_alpha = || sum f_alpha(s_qbar) Y_qbar / sum Y_qbar - f_alpha(s_0) ||_2 over
    the frames of one configuration.  s_est (F, 3) are the estimated DOAs s_qbar (grid points), Y (F,) their energies
    Y_qbar (eq. 5), s0 (3,) the true DOA.  Frames without a DOA (q = -1) are passed with Y = 0 (they carry no
    weight); a configuration whose weights sum to 0 has no estimate and returns nan."""
    f = MAPS[int(alpha)]
    Y = np.asarray(Y, dtype=np.float64)
    den = float(np.sum(Y))
    if den == 0.0:
        return float("nan")
    est = np.sum(f(np.asarray(s_est, dtype=np.float64)) * Y[:, None], axis=0) / den
    return float(np.linalg.norm(est - f(np.asarray(s0, dtype=np.float64))))


def rmse_from_indices(alpha: int, points: np.ndarray, q: np.ndarray, Y: np.ndarray, s0: np.ndarray) -> float:
    """rmse() with s_qbar = points[q] (q = -1: no DOA, weight 0)."""
    q = np.asarray(q)
    ok = q >= 0
    s_est = np.zeros((q.size, 3))
    s_est[ok] = np.asarray(points, dtype=np.float64)[q[ok]]
    return rmse(alpha, s_est, np.where(ok, Y, 0.0), s0)
