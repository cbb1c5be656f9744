"""SVD-PHAT oracle (§3, eqs. 10-15 and Algorithm 1), float64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Follows Algorithm 1 step by step:
offline 1 W, 2 SVD + rank rule, 3 normalised dictionary rows, 4 k-d tree; online 1 X, 2 Z and Z_hat,
3 nearest row (brute force and k-d tree), 4 Y_q_bar from the corresponding row of W.
"""
from __future__ import annotations

import numpy as np

from . import srpphat as srp
from .kdtree import KDTree


def rank_rule(sigma2_desc: np.ndarray, total: float, delta: float) -> int:
    """Eq. 11: smallest D with sum_{d<=D} sigma_d^2 >= (1 - delta) Tr{W W^H} (inclusive, reading R12)."""
    csum = np.cumsum(sigma2_desc)
    idx = np.nonzero(csum >= (1.0 - delta) * total)[0]
    return int(idx[0]) + 1 if idx.size else int(sigma2_desc.size)


def gram_pass(tau: np.ndarray, N: int, x: np.ndarray | None = None, chunk: int = 2048):
    """One pass over column chunks of W (eqs. 4, 8; W is never held whole):

      G = W W^H     (the Gram matrix of eq. 10: W = U S V^H  =>  W W^H = U S^2 U^H, so its eigenpairs are the
                     squared singular values and left singular vectors of W);
      total = Tr{W W^H} = sum |W|^2 (eq. 11's denominator, from W itself);
      WX = W x_f for every frame f of x, if x (F, PK) is given (eq. 9 before taking Re{}).

    G is accumulated by BLAS zherk and only its upper triangle is valid.  Returns (G, total, WX or None)."""
    from scipy.linalg import blas
    Q, P = tau.shape
    PK = P * (N // 2 + 1)
    G = np.zeros((Q, Q), dtype=np.complex128, order="F")
    WX = None if x is None else np.zeros((x.shape[0], Q), dtype=np.complex128)
    total = 0.0
    for c0 in range(0, PK, chunk):
        c1 = min(PK, c0 + chunk)
        Wc = srp.steering_cols(tau, N, c0, c1)
        G = blas.zherk(1.0, Wc, beta=1.0, c=G, trans=0, lower=0, overwrite_c=1)
        total += float(np.sum(Wc.real ** 2 + Wc.imag ** 2))
        if x is not None:
            WX += x[:, c0:c1] @ Wc.T
    return G, total, WX


def factors_from_gram(G: np.ndarray, total: float, delta: float, rank: int | None = None,
                      n_top: int | None = None) -> dict:
    """Alg. 1 offline steps 2-3 from the Gram matrix G = W W^H (upper triangle used).

    Eigenpairs of G by LAPACK (scipy.linalg.eigh; only the n_top largest when n_top < Q: eq. 11 needs only the
    leading sigma^2 because its denominator Tr{W W^H} is known exactly), descending; D by the rank rule eq. 11
    (P:140); U_D, S_D; R = U S (eq. 13) and the normalised rows R_hat.  Raises ValueError if the
    n_top leading eigenvalues do not reach (1 - delta) Tr{W W^H} (the caller asks for more)."""
    import scipy.linalg
    Q = G.shape[0]
    n = Q if n_top is None else min(Q, int(n_top))
    lam, Uall = scipy.linalg.eigh(G, lower=False, subset_by_index=[Q - n, Q - 1], driver="evr",
                                  check_finite=False)
    order = np.argsort(lam)[::-1]
    sigma2 = np.clip(lam[order], 0.0, None)
    if rank:
        D = int(rank)
    else:
        D = rank_rule(sigma2, total, delta)
        if n < Q and np.sum(sigma2) < (1.0 - delta) * total:
            raise ValueError(f"the {n} leading eigenvalues hold less than 1 - delta of Tr(WW^H): ask for more")
    U = Uall[:, order[:D]]
    S = np.sqrt(sigma2[:D])
    R = U * S[None, :]                                            # eq. 13: D = U S
    Rhat = R / np.linalg.norm(R, axis=1, keepdims=True)
    return dict(sigma2=sigma2, D=D, U=U, S=S, R=R, Rhat=Rhat, total=total, method="gram")


def svd_factors(tau: np.ndarray, N: int, delta: float = 1e-5, rank: int | None = None,
                method: str = "auto", chunk: int = 2048, n_top: int | None = None) -> dict:
    """Alg. 1 offline steps 1-3.

    method "svd": numpy/LAPACK SVD of the full W (eq. 10) - for small W.
    method "gram": eigen-decomposition of W W^H accumulated over column chunks of W (gram_pass +
                   factors_from_gram: same sigma^2 and U; V from V_D = W^H U_D S_D^{-1}), for W too large to
                   hold (cfg3-5).  Pinned against "svd" in tests.
    Returns dict(sigma2 (descending; all of them, or the n_top leading ones), D, U (Q,D), S (D,), V (PK,D),
                 R = U S (eq. 13), Rhat (rows / ||row||), total = Tr{W W^H} computed from W).
    """
    Q, P = tau.shape
    K = N // 2 + 1
    PK = P * K
    if method == "auto":
        method = "svd" if Q * PK <= 2.5e7 else "gram"
    if method == "svd":
        W = srp.steering_cols(tau, N, 0, PK)
        U, s, Vh = np.linalg.svd(W, full_matrices=False)
        sigma2 = s ** 2
        total = float(np.sum(np.abs(W) ** 2))
        D = rank if rank else rank_rule(sigma2, total, delta)
        U, S, V = U[:, :D], s[:D], Vh[:D].conj().T
        R = U * S[None, :]                                        # eq. 13: D = U S
        Rhat = R / np.linalg.norm(R, axis=1, keepdims=True)
        return dict(sigma2=sigma2, D=D, U=U, S=S, V=V, R=R, Rhat=Rhat, total=total, method=method)
    G, total, _ = gram_pass(tau, N, chunk=chunk)
    fac = factors_from_gram(G, total, delta, rank, n_top)
    del G
    U, S, D = fac["U"], fac["S"], fac["D"]
    V = np.empty((PK, D), dtype=np.complex128)
    for c0 in range(0, PK, chunk):
        c1 = min(PK, c0 + chunk)
        Wc = srp.steering_cols(tau, N, c0, c1)
        V[c0:c1] = (Wc.conj().T @ U) / S[None, :]
    fac["V"] = V
    return fac


def project(V: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Eq. 12: Z = V^H X.  x (F, PK) -> Z (F, D)."""
    return x @ V.conj()


def project_wx(fac: dict, WX: np.ndarray) -> np.ndarray:
    """Eq. 12 with the Gram-route V_D = W^H U_D S_D^{-1} substituted (eq. 10: U_D^H W = S_D V_D^H):
    Z_f = V_D^H x_f = S_D^{-1} U_D^H (W x_f).  WX (F, Q) = W x_f per frame (gram_pass) -> Z (F, D).  Used when
    V_D itself (PK x D) would cost a second pass over W (cfg3/cfg4 parity); pinned against project() in tests."""
    return (WX @ fac["U"].conj()) / fac["S"][None, :]


def search_scores(Rhat: np.ndarray, Zhat: np.ndarray) -> np.ndarray:
    """Re{D_hat_q . Z_hat} for all q (eq. 14 with normalised rows, reading R8): (F, Q)."""
    return np.real(Zhat @ Rhat.T)


def nearest_brute(Rhat: np.ndarray, Zhat: np.ndarray, tol: float = 1e-9) -> np.ndarray:
    """Eq. 15: argmin_q ||D_hat_q - Z_hat^H||^2 over all q, lowest index among near-ties (tol)."""
    out = np.empty(Zhat.shape[0], dtype=np.int64)
    for f in range(Zhat.shape[0]):
        d = np.sum(np.abs(Rhat - np.conj(Zhat[f])[None, :]) ** 2, axis=1)
        out[f] = int(np.argmax(d <= d.min() + tol))
    return out


def svd_localize(fac: dict, tau: np.ndarray, x: np.ndarray, N: int, use_tree: bool = False,
                 tree: KDTree | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Alg. 1 online steps 2-4.  Returns (q_bar int64 (-1 if degenerate), Y_q_bar float64)."""
    Z = project(fac["V"], x)
    nz = np.linalg.norm(Z, axis=1)
    dg = (nz == 0) | srp.degenerate(x)
    Zhat = Z / np.where(nz > 0, nz, 1.0)[:, None]
    if use_tree:
        tree = tree or KDTree(np.concatenate([fac["Rhat"].real, fac["Rhat"].imag], axis=1))
        q = np.array([tree.nearest_tie(np.concatenate([z.real, -z.imag])) for z in Zhat], dtype=np.int64)
    else:
        q = nearest_brute(fac["Rhat"], Zhat)
    score = np.empty(x.shape[0])
    for f in range(x.shape[0]):                                   # step 4: Y_q_bar from the row of W
        score[f] = float(np.real(srp.steering_rows(tau[q[f]:q[f] + 1], N)[0] @ x[f]))
    q[dg] = -1
    score[dg] = 0.0
    return q, score
