"""Pins of oracle/rmse.py (§4: f_1, f_2, f_3 and eq. results_rmse) — no GPU.

The mappings are pinned by closed-form values and by the array physics they encode: the paper maps a 1-D array's
estimates to an arc and a planar array's to a hemisphere because those arrays cannot tell the merged directions
apart.  So f_1 / f_2 must merge exactly the directions whose TDOAs (eq. 2, via the oracle's
tdoa_farfield, itself pinned) are identical for the Table 2 arrays, and nothing else.
"""
import json
import os

import numpy as np
import pytest

from oracle import rmse as R
from oracle import srpphat as srp

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "paper_table2_cm.json")) as _f:
    T2 = {k: np.asarray(v, dtype=np.float64) / 100.0 for k, v in json.load(_f).items() if not k.startswith("_")}
r2 = np.sqrt(0.5)


@pytest.mark.parametrize("s, want", [
    ((0, 0, 1), (0, 0, 1)),          # endfire up: elevation +90
    ((0, 0, -1), (0, 0, -1)),
    ((0, 1, 0), (1, 0, 0)),          # broadside: elevation 0
    ((-1, 0, 0), (1, 0, 0)),
    ((r2, 0, r2), (r2, 0, r2)),      # already on the arc
    ((0, -r2, -r2), (r2, 0, -r2)),   # elevation -45 from another azimuth
])
def test_f1_closed_form(s, want):
    """f_1(s) = [cos g, 0, sin g] with g = atan2(s_z, sqrt(s_x^2+s_y^2)): swapping atan2's arguments or
    using the azimuth instead of the elevation fails these."""
    assert np.allclose(R.f1(np.array(s, dtype=float)), want, atol=1e-15)


def test_f2_f3_closed_form():
    s = np.array([[0.3, -0.4, -0.866], [0.1, 0.2, 0.3]])
    assert np.allclose(R.f2(s), [[0.3, -0.4, 0.866], [0.1, 0.2, 0.3]], atol=0)
    assert np.array_equal(R.f3(s), s)


def _sphere(n, seed=0):
    v = np.random.default_rng(seed).normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def test_f1_merges_exactly_the_1d_array_ambiguity():
    """The Table 2 1-D array lies on the z axis: s and its rotation about z have identical TDOAs (eq. 2), and
    f_1 maps them to the same point; directions with different TDOAs stay apart."""
    mics = T2["1d"]
    s = _sphere(200, 1)
    phi = np.random.default_rng(2).uniform(0, 2 * np.pi, 200)
    c, sn = np.cos(phi), np.sin(phi)
    rot = np.stack([c * s[:, 0] - sn * s[:, 1], sn * s[:, 0] + c * s[:, 1], s[:, 2]], axis=1)
    t1, t2 = srp.tdoa_farfield(mics, s, 16000.0, 343.0), srp.tdoa_farfield(mics, rot, 16000.0, 343.0)
    assert np.allclose(t1, t2, atol=1e-12)
    assert np.allclose(R.f1(s), R.f1(rot), atol=1e-12)
    # different elevations -> different TDOAs and different f_1 images
    other = _sphere(200, 3)
    dt = np.abs(srp.tdoa_farfield(mics, other, 16000.0, 343.0) - t1).max(axis=1)
    df = np.linalg.norm(R.f1(other) - R.f1(s), axis=1)
    assert np.all((dt > 1e-6) == (df > 1e-9))


def test_f2_merges_exactly_the_planar_array_ambiguity():
    """The Table 2 2-D array lies in z = 0: s and its mirror (s_x, s_y, -s_z) have identical TDOAs, and f_2 maps
    both to the positive hemisphere; f_3 (3-D array) keeps them apart, as do that array's TDOAs."""
    s = _sphere(200, 4)
    mir = s * np.array([1.0, 1.0, -1.0])
    assert np.allclose(srp.tdoa_farfield(T2["2d"], s, 16000.0, 343.0),
                       srp.tdoa_farfield(T2["2d"], mir, 16000.0, 343.0), atol=1e-12)
    assert np.allclose(R.f2(s), R.f2(mir), atol=0)
    assert np.all(R.f2(s)[:, 2] >= 0)
    far = np.abs(s[:, 2]) > 1e-3
    assert np.all(np.abs(srp.tdoa_farfield(T2["3d"], s, 16000.0, 343.0)
                         - srp.tdoa_farfield(T2["3d"], mir, 16000.0, 343.0)).max(axis=1)[far] > 1e-6)
    assert np.all(np.linalg.norm(R.f3(s) - R.f3(mir), axis=1)[far] > 1e-3)


@pytest.mark.parametrize("alpha", [1, 2, 3])
def test_maps_keep_unit_vectors_and_are_idempotent(alpha):
    s = _sphere(100, 5)
    f = R.MAPS[alpha]
    assert np.allclose(np.linalg.norm(f(s), axis=1), 1.0, atol=1e-14)
    assert np.allclose(f(f(s)), f(s), atol=1e-14)


@pytest.mark.parametrize("alpha", [1, 2, 3])
def test_rmse_special_cases(alpha):
    """Eq. results_rmse: exact estimates -> 0; one frame -> the distance of the mapped points; the energy
    weights form a weighted mean (weights 1 and 3 -> 1/4, 3/4) and only their ratios matter."""
    s0 = np.array([0.48, 0.6, 0.64])
    a, b = np.array([0.0, 0.6, 0.8]), np.array([0.8, -0.6, 0.0])
    f = R.MAPS[alpha]
    assert R.rmse(alpha, np.stack([s0, s0, s0]), np.array([1.0, 2.0, 5.0]), s0) == pytest.approx(0.0, abs=1e-15)
    assert R.rmse(alpha, a[None], np.array([7.0]), s0) == pytest.approx(np.linalg.norm(f(a) - f(s0)), abs=1e-15)
    want = np.linalg.norm(0.25 * f(a) + 0.75 * f(b) - f(s0))
    assert R.rmse(alpha, np.stack([a, b]), np.array([1.0, 3.0]), s0) == pytest.approx(want, abs=1e-15)
    assert R.rmse(alpha, np.stack([a, b]), np.array([10.0, 30.0]), s0) == pytest.approx(want, abs=1e-15)


def test_rmse_ambiguity_is_not_an_error():
    """A planar array's mirror estimate and a linear array's rotated estimate are not localisation errors."""
    s0 = np.array([0.48, 0.6, 0.64])
    assert R.rmse(2, (s0 * [1, 1, -1])[None], np.ones(1), s0) == pytest.approx(0.0, abs=1e-15)
    rot = np.array([-0.6, 0.48, 0.64])
    assert R.rmse(1, rot[None], np.ones(1), s0) == pytest.approx(0.0, abs=1e-15)
    assert R.rmse(3, rot[None], np.ones(1), s0) > 0.5


def test_rmse_from_indices_skips_frames_without_doa():
    pts = np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0]])
    s0 = np.array([0.0, 0.0, 1.0])
    assert R.rmse_from_indices(3, pts, np.array([0, -1]), np.array([2.0, 5.0]), s0) == pytest.approx(0.0)
    assert np.isnan(R.rmse_from_indices(3, pts, np.array([-1]), np.array([5.0]), s0))
