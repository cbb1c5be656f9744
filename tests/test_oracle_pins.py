"""Pins of the float64 oracle against what the paper and mathematics fix (no GPU).

Each test names the PAPER.md passage (P:n) or the independent fact it checks.  None of them retypes the
oracle's own formula: they use closed forms, paper numbers (tests/golden/), textbook routines (numpy.fft),
independent algebraic identities, brute force, and physics-level injections through workloads/scenes.py.
"""
import json
import os

import numpy as np
import pytest

from oracle import srpphat as srp
from oracle import svdphat as svd
from oracle.kdtree import KDTree
from workloads import geometry as G
from workloads import scenes as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _paper_mics(name):
    return np.asarray(_gold("paper_table2_cm.json")[name], dtype=np.float64) / 100.0


T1 = _gold("paper_table1.json")
FS, C = float(T1["fs"]), float(T1["c"])


# ------------------------------------------------------------------ eq. 1 / eq. 2
def test_tdoa_farfield_closed_form():
    mics = _paper_mics("1d")
    tau = srp.tdoa_farfield(mics, np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0], [0.0, 0.0, -1.0]]), FS, C)
    p = srp.pairs(7).index((0, 6))
    assert tau[0, p] == pytest.approx(16000.0 / 343.0 * 0.10, abs=1e-12)   # 4.664723 samples
    assert tau[1, p] == pytest.approx(0.0, abs=1e-15)                      # orthogonal to the baseline
    assert np.allclose(tau[2], -tau[0], atol=0)                            # antisymmetric in u
    # non-unit s_q is normalised by eq. 2 itself
    tau2 = srp.tdoa_farfield(mics, np.array([[0.0, 0.0, 7.5]]), FS, C)
    assert np.allclose(tau2[0], tau[0], atol=1e-13)


def test_tdoa_bound_and_pair_antisymmetry():
    rng = np.random.default_rng(0)
    mics = rng.uniform(-0.1, 0.1, (6, 3))
    u = rng.standard_normal((200, 3))
    for fld, pts in (("far", u), ("near", u * 0.7)):
        tau = srp.tdoa(mics, pts, FS, C, fld)
        for p, (i, j) in enumerate(srp.pairs(6)):
            lim = FS / C * np.linalg.norm(mics[i] - mics[j])
            assert np.all(np.abs(tau[:, p]) <= lim * (1 + 1e-12))
        # swapping the mic order of the array reverses each pair's sign
        tau_sw = srp.tdoa(mics[::-1], pts, FS, C, fld)
        P = len(srp.pairs(6))
        for p, (i, j) in enumerate(srp.pairs(6)):
            q = srp.pairs(6).index((5 - j, 5 - i))
            assert np.allclose(tau_sw[:, q], -tau[:, p], atol=1e-12)
        assert P == 15


def test_tdoa_exact_closed_form_and_farfield_limit():
    mics = _paper_mics("1d")
    p = srp.pairs(7).index((0, 6))
    tau = srp.tdoa_exact(mics, np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0]]), FS, C)
    assert tau[0, p] == pytest.approx(16000.0 / 343.0 * (1.05 - 0.95), abs=1e-12)
    assert tau[1, p] == pytest.approx(0.0, abs=1e-12)
    # far-field convergence: at R = 100 * aperture, |tau_exact - tau_far| < 0.01 samples
    rng = np.random.default_rng(1)
    u = rng.standard_normal((100, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    R = 100 * 0.10
    d = srp.tdoa_exact(mics, R * u, FS, C) - srp.tdoa_farfield(mics, u, FS, C)
    assert np.max(np.abs(d)) < 0.01


# ------------------------------------------------------------------ STFT
def test_stft_equals_numpy_rfft():
    rng = np.random.default_rng(2)
    fr = rng.standard_normal((3, 4, 64))
    X = srp.stft(fr)
    ref = np.fft.rfft(fr * np.sin(np.pi * (np.arange(64) + 0.5) / 64), axis=-1)
    assert np.max(np.abs(X - ref)) < 1e-11 * np.max(np.abs(ref))


def test_stft_tone_and_dc():
    N = 512
    n = np.arange(N)
    X = srp.stft(np.cos(2 * np.pi * 16 * n / N)[None, None, :])[0, 0]
    assert int(np.argmax(np.abs(X))) == 16
    Xdc = np.abs(srp.stft(np.ones((1, 1, N)))[0, 0])
    assert set(np.argsort(Xdc)[-2:]) == {0, 1}          # sine-window main lobe


def test_framing_counts():
    assert srp.frame_count(32000, 512, 256) == 124      # BJ.cfg1 "~124 frames"
    assert srp.frame_count(960000, 512, 256) == 3749    # BJ.cfg2 "~3750 frames"
    assert srp.frame_count(511, 512, 256) == 0
    assert srp.frame_count(512, 512, 256) == 1
    a = np.arange(2 * 1000, dtype=np.float32).reshape(2, 1000)
    fr = srp.extract_frames(a, srp.frame_count(1000, 64, 32), 2, 64, 1000, 32)
    assert fr.shape == (30, 2, 64)
    assert fr[7, 1, 5] == 1000 + 7 * 32 + 5


# ------------------------------------------------------------------ eq. 3 / eq. 7
def test_cross_spectrum_conventions():
    rng = np.random.default_rng(3)
    K, N = 33, 64
    Xi = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    k = np.arange(K)
    d = 3
    X = np.stack([Xi, 2.5 * Xi * np.exp(-2j * np.pi * k * d / N), Xi, np.zeros(K)])[None]
    x = srp.cross_spectrum(X).reshape(6, K)
    P = srp.pairs(4)
    assert np.allclose(x[P.index((0, 2))], 1.0, atol=1e-15)                          # identical channels
    assert np.allclose(x[P.index((0, 1))], np.exp(2j * np.pi * k * d / N), atol=1e-14)  # +2 pi k d / N
    assert np.all(x[P.index((0, 3))] == 0) and np.all(x[P.index((2, 3))] == 0)        # zero guard
    assert np.allclose(np.abs(x[[P.index((0, 1)), P.index((0, 2)), P.index((1, 2))]]), 1.0, atol=1e-14)
    # pair-major with bins inner (eq. 7)
    xf = srp.cross_spectrum(X)[0]
    assert xf[P.index((0, 1)) * K + 5] == x[P.index((0, 1)), 5]


# ------------------------------------------------------------------ W, Y (eqs. 4, 5, 8, 9)
def _small_case(level=2, N=64, name="3d"):
    mics = _paper_mics(name)
    grid = G.icosphere(level)
    return mics, grid, srp.tdoa_farfield(mics, grid, FS, C), N


def test_steering_frobenius_and_self_match():
    mics, grid, tau, N = _small_case(4, 256, "3d")
    K = N // 2 + 1
    Q, P = tau.shape
    tot = 0.0
    for q0 in range(0, Q, 512):
        W = srp.steering_rows(tau[q0:q0 + 512], N)
        tot += np.sum(np.abs(W) ** 2)
    assert tot == pytest.approx(Q * P * K, rel=1e-12)        # 2562*21*129 = 6,940,458 (|W| = 1)
    assert Q * P * K == 6940458
    assert srp.steering_rows(tau[:1], N)[0, :K].real[0] == 1.0   # k = 0 column is 1
    qs = np.array([5, 777, 2000])
    x = np.conj(srp.steering_rows(tau[qs], N))
    Y = srp.srp_energy(tau, x, N)
    for r, q in enumerate(qs):
        assert Y[r, q] == pytest.approx(P * K, rel=1e-12)
        assert np.all(Y[r] <= P * K * (1 + 1e-12))
    qb, _ = srp.argmax_tie(Y)
    assert list(qb) == list(qs)


def test_srp_energy_equals_literal_eq5():
    rng = np.random.default_rng(4)
    mics, grid, tau, N = _small_case(1, 32)
    X = rng.standard_normal((2, 7, N // 2 + 1)) + 1j * rng.standard_normal((2, 7, N // 2 + 1))
    X[1, 3, 4] = 0.0
    x = srp.cross_spectrum(X)
    Y = srp.srp_energy(tau, x, N)
    for f in range(2):
        for q in (0, 17, 41):
            assert Y[f, q] == pytest.approx(srp.srp_energy_direct(tau[q], X[f], N), rel=1e-11, abs=1e-10)


def test_srp_energy_delay_and_sum_identity():
    """Independent O(QMK) formula: tau_qij = d_qi - d_qj gives
    Y_q = 1/2 sum_k (|sum_m e_m[k] exp(+j2pi k d_qm / N)|^2 - n_k), n_k = #non-zero phasors at bin k."""
    rng = np.random.default_rng(5)
    mics, grid, tau, N = _small_case(2, 64)
    K = N // 2 + 1
    fr = rng.standard_normal((3, 7, N))
    fr[2, 4] = 0.0                                           # one silent channel
    X = srp.stft(fr)
    x = srp.cross_spectrum(X)
    Y = srp.srp_energy(tau, x, N)
    delay = -(FS / C) * grid @ mics.T                        # (Q, M) arrival delays, any common offset
    e = np.where(np.abs(X) > 0, X / np.where(np.abs(X) > 0, np.abs(X), 1), 0)
    k = np.arange(K)
    for f in range(3):
        nk = np.sum(np.abs(e[f]) > 0, axis=0)
        a = e[f][None, :, :] * np.exp(2j * np.pi * k[None, None, :] * delay[:, :, None] / N)   # (Q, M, K)
        ds = 0.5 * np.sum(np.abs(a.sum(axis=1)) ** 2 - nk[None, :], axis=1)
        assert np.max(np.abs(ds - Y[f])) < 1e-9 * np.max(np.abs(Y[f]))


def test_injection_returns_grid_point_3d():
    """Noiseless fractional-delay plane waves from grid directions (workloads.scenes physics) -> q (sign pin)."""
    mics, grid, tau, N = _small_case(3, 256, "3d")
    rng = np.random.default_rng(6)
    qs = rng.choice(grid.shape[0], 12, replace=False)
    fr = np.stack([S.plane_wave_stream(rng, mics, FS, C, N, grid[q], 300.0) for q in qs])
    x = srp.frames_to_x(fr)
    qb, _ = srp.srp_localize(tau, x, N)
    assert list(qb) == list(qs)
    # flipping the sign of eq. 4 would point at the antipode
    Yflip = srp.srp_energy(-tau, x, N)
    anti = np.argmin(grid @ grid[qs].T, axis=0)
    assert list(np.argmax(Yflip, axis=1)) == list(anti)


def test_injection_planar_twin_lowest_index():
    mics, grid, tau, N = _small_case(3, 256, "2d")
    rng = np.random.default_rng(7)
    mirror = {i: int(np.argmin(np.linalg.norm(grid - grid[i] * [1, 1, -1], axis=1))) for i in range(len(grid))}
    qs = [q for q in rng.choice(grid.shape[0], 40, replace=False) if mirror[q] != q][:8]
    fr = np.stack([S.plane_wave_stream(rng, mics, FS, C, N, grid[q], 300.0) for q in qs])
    qb, _ = srp.srp_localize(tau, srp.frames_to_x(fr), N)
    assert list(qb) == [min(q, mirror[q]) for q in qs]


def test_degenerate_frame():
    mics, grid, tau, N = _small_case(1, 32)
    fr = np.zeros((2, 7, N))
    fr[1, 0] = np.random.default_rng(8).standard_normal(N)     # only one live channel: X vector is 0
    q, s = srp.srp_localize(tau, srp.frames_to_x(fr), N)
    assert list(q) == [-1, -1] and list(s) == [0.0, 0.0]


# ------------------------------------------------------------------ rank rule (eq. 11) vs the paper's gains
@pytest.mark.parametrize("name", ["1d", "2d", "3d"])
def test_rank_rule_reproduces_paper_gains(name):
    gains = _gold("paper_gains.json")
    mics = _paper_mics(name)
    grid = G.icosphere(4)
    assert grid.shape[0] == T1["Q"]
    tau = srp.tdoa_farfield(mics, grid, FS, C)
    fac = svd.svd_factors(tau, T1["N"], gains["delta"], method="svd")
    assert fac["total"] == pytest.approx(grid.shape[0] * 21 * (T1["N"] // 2 + 1), rel=1e-12)
    assert round(T1["Q"] / fac["D"]) == gains["gain"][name]
    # minimality: D-1 violates eq. 11
    s2 = fac["sigma2"]
    assert np.sum(s2[:fac["D"]]) >= (1 - gains["delta"]) * fac["total"]
    assert np.sum(s2[:fac["D"] - 1]) < (1 - gains["delta"]) * fac["total"]


def test_rank_one_toy():
    tau = np.zeros((5, 1))                      # identical rows
    fac = svd.svd_factors(tau, 2, 1e-3, method="svd")
    assert fac["D"] == 1


def test_svd_and_gram_routes_agree():
    mics, grid, tau, N = _small_case(2, 64, "2d")
    a = svd.svd_factors(tau, N, 1e-5, method="svd")
    b = svd.svd_factors(tau, N, 1e-5, method="gram", chunk=100)
    assert a["D"] == b["D"]
    n = min(len(a["sigma2"]), 40)
    assert np.allclose(a["sigma2"][:n], b["sigma2"][:n], rtol=1e-9, atol=1e-9 * a["sigma2"][0])
    rng = np.random.default_rng(9)
    x = srp.frames_to_x(rng.standard_normal((4, 7, N)))
    for f in (a, b):
        f["_s"] = svd.search_scores(f["Rhat"], svd.project(f["V"], x) /
                                    np.linalg.norm(svd.project(f["V"], x), axis=1, keepdims=True))
    assert np.max(np.abs(a["_s"] - b["_s"])) < 1e-9


def test_full_rank_svd_equals_srp():
    mics, grid, tau, N = _small_case(2, 64, "3d")
    rng = np.random.default_rng(10)
    fac = svd.svd_factors(tau, N, 1e-14, method="svd")
    u = rng.standard_normal((30, 3))
    fr = np.stack([S.plane_wave_stream(rng, mics, FS, C, N, uu / np.linalg.norm(uu), 5.0) for uu in u])
    x = srp.frames_to_x(fr)
    q1, s1 = srp.srp_localize(tau, x, N)
    q2, s2 = svd.svd_localize(fac, tau, x, N)
    assert list(q1) == list(q2)
    assert np.allclose(s1, s2, rtol=1e-10)


def test_eq15_distance_identity():
    rng = np.random.default_rng(11)
    a = rng.standard_normal((1000, 9)) + 1j * rng.standard_normal((1000, 9))
    b = rng.standard_normal((1000, 9)) + 1j * rng.standard_normal((1000, 9))
    a /= np.linalg.norm(a, axis=1, keepdims=True)
    b /= np.linalg.norm(b, axis=1, keepdims=True)
    lhs = np.real(np.sum(a * b, axis=1))
    rhs = 1 - 0.5 * np.sum(np.abs(a - np.conj(b)) ** 2, axis=1)
    assert np.max(np.abs(lhs - rhs)) < 1e-12


def test_svd_injection_returns_grid_point():
    mics, grid, tau, N = _small_case(3, 256, "3d")
    fac = svd.svd_factors(tau, N, 1e-5, method="svd")
    rng = np.random.default_rng(12)
    qs = rng.choice(grid.shape[0], 10, replace=False)
    fr = np.stack([S.plane_wave_stream(rng, mics, FS, C, N, grid[q], 300.0) for q in qs])
    x = srp.frames_to_x(fr)
    q, s = svd.svd_localize(fac, tau, x, N)
    assert list(q) == list(qs)
    qt, _ = svd.svd_localize(fac, tau, x, N, use_tree=True)
    assert list(qt) == list(qs)


# ------------------------------------------------------------------ k-d tree == brute force
@pytest.mark.parametrize("n,dim", [(12, 2), (42, 4), (162, 16), (300, 3)])
def test_kdtree_equals_brute_force(n, dim):
    rng = np.random.default_rng(n + dim)
    pts = rng.standard_normal((n, dim))
    pts[n // 2] = pts[3]                              # exact duplicates / twins
    pts[n - 1] = pts[0]
    pts = np.round(pts, 2)                            # many exact distance ties
    t = KDTree(pts, leaf_size=4)
    for _ in range(200):
        qv = np.round(rng.standard_normal(dim), 1) if _ % 2 else pts[rng.integers(n)]
        d = np.array([float((p - qv) @ (p - qv)) for p in pts])   # same per-point arithmetic as the tree
        brute = int(np.argmin(d))                     # numpy argmin returns the lowest index on ties
        i, d2 = t.nearest(qv)
        assert i == brute and d2 == d[brute]


def test_kdtree_singleton_and_self_query():
    t = KDTree(np.array([[1.0, 2.0]]))
    assert t.nearest(np.array([5.0, -3.0]))[0] == 0
    pts = np.random.default_rng(13).standard_normal((100, 6))
    t = KDTree(pts)
    for i in range(100):
        assert t.nearest(pts[i]) == (i, 0.0)


def test_topk_two_sources_injection():
    """Two noiseless plane waves from grid points far apart -> the two strongest separated peaks are those points;
    k = 1 equals the plain argmax."""
    mics, grid, tau, N = _small_case(3, 256, "3d")
    rng = np.random.default_rng(14)
    reps = srp.steering_classes(tau)
    assert len(reps) == len(grid)                       # 3-D array: no twins
    frames, truth = [], []
    for _ in range(6):
        while True:
            a, b = rng.choice(len(grid), 2, replace=False)
            if np.degrees(np.arccos(grid[a] @ grid[b])) > 110:
                break
        sig = S.plane_wave_stream(rng, mics, FS, C, N, grid[a], 300.0) + \
            S.plane_wave_stream(rng, mics, FS, C, N, grid[b], 300.0)
        frames.append(sig)
        truth.append({int(a), int(b)})
    x = srp.frames_to_x(np.stack(frames))
    Y = srp.srp_energy(tau, x, N)
    top = srp.topk_peaks(Y, grid, reps, 2, 60.0)     # 10 cm aperture: broad main lobes
    for f in range(len(truth)):                         # each source within one level-3 grid spacing (~8 deg)
        for t in truth[f]:
            assert min(np.degrees(np.arccos(np.clip(grid[q] @ grid[t], -1, 1))) for q in top[f]) < 10.0
    q1, _ = srp.argmax_tie(Y)
    assert list(srp.topk_peaks(Y, grid, reps, 1, 25.0)[:, 0]) == list(q1)


def test_steering_classes_planar():
    mics, grid, tau, N = _small_case(2, 64, "2d")
    reps = srp.steering_classes(tau)
    mirror = np.array([int(np.argmin(np.linalg.norm(grid - g * [1, 1, -1], axis=1))) for g in grid])
    assert sorted(reps.tolist()) == sorted(set(np.minimum(np.arange(len(grid)), mirror).tolist()))


# ------------------------------------------------------------------ DESIGN.md R22: antipodal folding
def _antipode_index(grid):
    key = {r.tobytes(): i for i, r in enumerate(grid + 0.0)}
    return np.array([key[((-r) + 0.0).tobytes()] for r in grid])


def test_antipodal_fold_identity():
    """Eq. 2 is odd in s_q, so on a centrally symmetric grid tau(-s) = -tau(s) bitwise, W_{q'} = conj(W_q) (eq. 4) and
    eq. 9 for the pair follows from two real half products: Y_q = a - b, Y_q' = a + b with a = Re W_q . Re X and
    b = Im W_q . Im X (the GPU's fold rows).  Checked against the oracle's complex BLAS product."""
    rng = np.random.default_rng(22)
    mics = rng.uniform(-0.06, 0.06, (7, 3))
    grid = G.icosphere(2)
    N = 128
    tau = srp.tdoa_farfield(mics, grid, FS, C)
    anti = _antipode_index(grid)
    assert np.all(anti != np.arange(len(grid)))
    for q in range(len(grid)):
        assert np.array_equal(tau[anti[q]], -tau[q] + 0.0)
    W = srp.steering_rows(tau, N)
    assert np.max(np.abs(W[anti] - np.conj(W))) < 1e-12
    x = srp.frames_to_x(rng.standard_normal((5, 7, N)))
    Y = srp.srp_energy(tau, x, N)
    a = np.real(W) @ np.real(x).T          # (Q, F)
    b = np.imag(W) @ np.imag(x).T
    scale = np.max(np.abs(Y))
    assert np.max(np.abs((a - b).T - Y)) < 1e-10 * scale
    assert np.max(np.abs((a + b).T - Y[:, anti])) < 1e-10 * scale


def test_symmetric_grid_gram_is_real():
    """With W_{q'} = conj(W_q) for every q, conj(W) = Pi W for the antipode permutation Pi, so W^H W is real and
    T W (rows sqrt2 Re W_q, sqrt2 Im W_q per antipodal pair) is a real matrix with W's singular values: the SVD of
    eq. 10 has a real V (R22, the GPU's real-V projection)."""
    rng = np.random.default_rng(23)
    mics = rng.uniform(-0.06, 0.06, (5, 3))
    grid = G.icosphere(2)
    N = 64
    tau = srp.tdoa_farfield(mics, grid, FS, C)
    W = srp.steering_rows(tau, N)
    Gr = W.conj().T @ W
    assert np.max(np.abs(Gr.imag)) < 1e-9 * np.max(np.abs(Gr))
    anti = _antipode_index(grid)
    prim = [q for q in range(len(grid)) if q < anti[q]]
    Wt = np.concatenate([np.sqrt(2) * W[prim].real, np.sqrt(2) * W[prim].imag])
    s_c = np.linalg.svd(W, compute_uv=False)
    s_r = np.linalg.svd(Wt, compute_uv=False)
    assert np.allclose(s_c, s_r, rtol=1e-9, atol=1e-9 * s_c[0])


# ------------------------------------------------------------------ Gram route of eq. 10 (cfg3/cfg4 parity path)
def test_gram_pass_top_subset_and_project_wx():
    """The one-pass Gram route used at headline size: zherk Gram of the column chunks equals W W^H, W x per frame
    equals the full product, the n_top-subset eigensolve gives LAPACK-SVD's D, sigma^2 and search scores (eq. 14),
    and Z from W x (V_D^H = S^{-1} U^H W, eq. 10) equals Z = V^H x from the SVD's own V (eq. 12)."""
    mics, grid, tau, N = _small_case(2, 64, "3d")
    rng = np.random.default_rng(31)
    x = srp.frames_to_x(rng.standard_normal((6, 7, N)))
    a = svd.svd_factors(tau, N, 1e-5, method="svd")
    G_, total, WX = svd.gram_pass(tau, N, x, chunk=97)
    W = srp.steering_cols(tau, N, 0, tau.shape[1] * (N // 2 + 1))
    assert np.max(np.abs(np.triu(G_) - np.triu(W @ W.conj().T))) < 1e-10 * np.abs(G_).max()
    assert np.max(np.abs(WX - x @ W.T)) < 1e-10 * np.abs(WX).max()
    assert total == pytest.approx(grid.shape[0] * 21 * (N // 2 + 1), rel=1e-12)
    full = svd.factors_from_gram(G_, total, 1e-5)
    top = svd.factors_from_gram(G_, total, 1e-5, n_top=a["D"] + 5)
    assert a["D"] == full["D"] == top["D"]
    n = a["D"] + 5
    assert np.allclose(top["sigma2"][:n], a["sigma2"][:n], rtol=1e-9, atol=1e-9 * a["sigma2"][0])
    assert np.allclose(full["sigma2"][:n], a["sigma2"][:n], rtol=1e-9, atol=1e-9 * a["sigma2"][0])
    Za = svd.project(a["V"], x)
    Zt = svd.project_wx(top, WX)
    sa = svd.search_scores(a["Rhat"], Za / np.linalg.norm(Za, axis=1, keepdims=True))
    st = svd.search_scores(top["Rhat"], Zt / np.linalg.norm(Zt, axis=1, keepdims=True))
    assert np.max(np.abs(sa - st)) < 1e-9
    assert np.allclose(np.linalg.norm(Za, axis=1), np.linalg.norm(Zt, axis=1), rtol=1e-10)
    with pytest.raises(ValueError):                # too few eigenpairs to reach (1 - delta) of the trace
        svd.factors_from_gram(G_, total, 1e-5, n_top=a["D"] - 1)


def test_gram_route_v_is_orthonormal():
    """Eq. 10: V_D has orthonormal columns (V^H V = I_D) and spans the same subspace as LAPACK's V (principal
    angles 0: the singular values of V_svd^H V_gram are all 1)."""
    mics, grid, tau, N = _small_case(2, 64, "2d")
    a = svd.svd_factors(tau, N, 1e-5, method="svd")
    b = svd.svd_factors(tau, N, 1e-5, method="gram", chunk=64)
    for f in (a, b):
        V = f["V"]
        assert np.max(np.abs(V.conj().T @ V - np.eye(f["D"]))) < 1e-10
    cosines = np.linalg.svd(a["V"].conj().T @ b["V"], compute_uv=False)
    assert np.min(cosines) > 1 - 1e-10


# ------------------------------------------------------------------ NEXT-3: binary TF masks
def test_tf_mask_identity_degenerate_and_delay_and_sum():
    """apply_tf_mask: an all-kept mask is the identity; a frame with every bin masked is degenerate (R4: q = -1);
    and the masked SRP power equals the independent delay-and-sum formula summed over the kept bins only:
    Y_q = 1/2 sum_{k kept} (|sum_m e_m[k] exp(+j2pi k d_qm / N)|^2 - n_k)."""
    rng = np.random.default_rng(41)
    mics, grid, tau, N = _small_case(2, 64)
    K, M = N // 2 + 1, 7
    P = M * (M - 1) // 2
    fr = rng.standard_normal((3, M, N))
    X = srp.stft(fr)
    x = srp.cross_spectrum(X)
    assert np.array_equal(srp.apply_tf_mask(x, P, np.ones((3, K), bool)), x)
    keep = rng.random((3, K)) < 0.6
    keep[1] = False
    xm = srp.apply_tf_mask(x, P, keep)
    q, s = srp.srp_localize(tau, xm, N)
    assert q[1] == -1 and s[1] == 0.0
    Y = srp.srp_energy(tau, xm, N)
    delay = -(FS / C) * grid @ mics.T
    e = np.where(np.abs(X) > 0, X / np.where(np.abs(X) > 0, np.abs(X), 1), 0)
    k = np.arange(K)
    for f in (0, 2):
        kk = k[keep[f]]
        ef = e[f][:, keep[f]]
        nk = np.sum(np.abs(ef) > 0, axis=0)
        a = ef[None, :, :] * np.exp(2j * np.pi * kk[None, None, :] * delay[:, :, None] / N)
        ds = 0.5 * np.sum(np.abs(a.sum(axis=1)) ** 2 - nk[None, :], axis=1)
        assert np.max(np.abs(ds - Y[f])) < 1e-9 * np.max(np.abs(Y[f]))
