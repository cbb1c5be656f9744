"""Property-based pins of the oracle (hypothesis, CPU, small random problems):

* svd and gram routes give the same D and the same search scores (eq. 10 vs W W^H);
* at full numerical rank SVD-PHAT returns SRP-PHAT's DOA (eq. 15 with D = rank);
* the k-d tree equals brute force on random point sets with duplicates;
* Y_q <= P(N/2+1) and the delay-and-sum form equals eq. 5 for random arrays, both field models (eqs. 1-2).
"""
import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import srpphat as srp
from oracle import svdphat as svd
from oracle.kdtree import KDTree
from workloads import geometry as G

FS, C = 16000.0, 343.0


def _setup(seed, M, N, level, field):
    rng = np.random.default_rng(seed)
    mics = rng.uniform(-0.06, 0.06, (M, 3))
    pts = G.icosphere(level)
    if field == "near":
        pts = pts * 0.8 + rng.uniform(-0.1, 0.1, 3)
    return rng, mics, pts, srp.tdoa(mics, pts, FS, C, field)


@settings(max_examples=12, deadline=None)
@given(seed=st.integers(0, 10_000), M=st.integers(2, 6), N=st.sampled_from([16, 32, 64]),
       level=st.integers(0, 2), field=st.sampled_from(["far", "near"]))
def test_srp_bound_and_delay_and_sum(seed, M, N, level, field):
    rng, mics, pts, tau = _setup(seed, M, N, level, field)
    fr = rng.standard_normal((3, M, N))
    X = srp.stft(fr)
    x = srp.cross_spectrum(X)
    Y = srp.srp_energy(tau, x, N)
    K = N // 2 + 1
    P = M * (M - 1) // 2
    assert np.all(Y <= P * K * (1 + 1e-12))
    if field == "far":
        delay = -(FS / C) * (pts / np.linalg.norm(pts, axis=1, keepdims=True)) @ mics.T
    else:
        delay = (FS / C) * np.linalg.norm(pts[:, None, :] - mics[None, :, :], axis=2)
    e = srp.phat_phasors(X)
    k = np.arange(K)
    for f in range(3):
        nk = np.sum(np.abs(e[f]) > 0, axis=0)
        a = e[f][None] * np.exp(2j * np.pi * k[None, None, :] * delay[:, :, None] / N)
        ds = 0.5 * np.sum(np.abs(a.sum(axis=1)) ** 2 - nk[None, :], axis=1)
        assert np.max(np.abs(ds - Y[f])) <= 1e-9 * max(1.0, np.max(np.abs(Y[f])))


@settings(max_examples=10, deadline=None)
@given(seed=st.integers(0, 10_000), M=st.integers(3, 6), N=st.sampled_from([32, 64]), level=st.integers(1, 2))
def test_svd_routes_and_full_rank(seed, M, N, level):
    rng, mics, pts, tau = _setup(seed, M, N, level, "far")
    a = svd.svd_factors(tau, N, 1e-4, method="svd")
    b = svd.svd_factors(tau, N, 1e-4, method="gram", chunk=37)
    assert a["D"] == b["D"]
    x = srp.frames_to_x(rng.standard_normal((4, M, N)))
    sa = svd.search_scores(a["Rhat"], svd.project(a["V"], x) / np.linalg.norm(svd.project(a["V"], x), axis=1,
                                                                               keepdims=True))
    sb = svd.search_scores(b["Rhat"], svd.project(b["V"], x) / np.linalg.norm(svd.project(b["V"], x), axis=1,
                                                                               keepdims=True))
    assert np.max(np.abs(sa - sb)) < 1e-8
    full = svd.svd_factors(tau, N, 1e-15, method="svd")
    q1, s1 = srp.srp_localize(tau, x, N)
    q2, s2 = svd.svd_localize(full, tau, x, N)
    Y = srp.srp_energy(tau, x, N)
    for f in range(4):       # equal, or an exact twin / near-tie of the SRP power
        assert q1[f] == q2[f] or abs(Y[f, q1[f]] - Y[f, q2[f]]) <= 1e-9 * abs(Y[f, q1[f]])


@settings(max_examples=25, deadline=None)
@given(seed=st.integers(0, 10_000), n=st.integers(1, 120), dim=st.integers(1, 9), leaf=st.integers(1, 17))
def test_kdtree_matches_brute_force(seed, n, dim, leaf):
    rng = np.random.default_rng(seed)
    pts = np.round(rng.standard_normal((n, dim)), 1)
    if n > 3:
        pts[rng.integers(n)] = pts[0]
    t = KDTree(pts, leaf_size=leaf)
    for _ in range(20):
        q = np.round(rng.standard_normal(dim), 1)
        d = np.array([float((p - q) @ (p - q)) for p in pts])
        i, d2 = t.nearest(q)
        assert i == int(np.argmin(d)) and d2 == d[i]
        assert t.nearest_tie(q) == min(np.nonzero(d <= d.min() + 1e-9)[0])
