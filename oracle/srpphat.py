"""SRP-PHAT oracle (§2, eqs. 1-6; §3 eqs. 7-9), float64, plain and slow on purpose.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  It shares
no code with the CUDA path (paper_1811_11785_b200/) and never imports it.

Each function cites the passage it follows (`P:n` = /root/reference/PAPER.md line n).  Readings of silent or
ambiguous passages are the `R*` items of DESIGN.md.
"""
from __future__ import annotations

import numpy as np


# ---------------------------------------------------------------- geometry (§2, eqs. 1-2)
def pairs(M: int) -> list[tuple[int, int]]:
    """Microphone pairs (i, j), i < j, in the order of eq. 5's double sum: (0,1),(0,2),...,(M-2,M-1)."""
    return [(i, j) for i in range(M) for j in range(i + 1, M)]


def tdoa_farfield(mics: np.ndarray, dirs: np.ndarray, fs: float, c: float) -> np.ndarray:
    """Eq. 2: tau_{q,i,j} = (fs/c) (r_j - r_i) . s_q / ||s_q||, in samples.  Returns (Q, P)."""
    s = dirs / np.linalg.norm(dirs, axis=1, keepdims=True)
    M = mics.shape[0]
    tau = np.empty((dirs.shape[0], M * (M - 1) // 2))
    for p, (i, j) in enumerate(pairs(M)):
        tau[:, p] = (fs / c) * (s @ (mics[j] - mics[i]))
    return tau


def tdoa_exact(mics: np.ndarray, pts: np.ndarray, fs: float, c: float) -> np.ndarray:
    """Eq. 1: tau_{q,i,j} = (fs/c) (||s_q - r_i|| - ||s_q - r_j||), in samples.  Returns (Q, P)."""
    M = mics.shape[0]
    tau = np.empty((pts.shape[0], M * (M - 1) // 2))
    for p, (i, j) in enumerate(pairs(M)):
        tau[:, p] = (fs / c) * (np.linalg.norm(pts - mics[i], axis=1) - np.linalg.norm(pts - mics[j], axis=1))
    return tau


def tdoa(mics, pts, fs, c, field: str) -> np.ndarray:
    return tdoa_farfield(mics, pts, fs, c) if field == "far" else tdoa_exact(mics, pts, fs, c)


# ---------------------------------------------------------------- framing + STFT (§2)
def frame_count(L: int, N: int, hop: int) -> int:
    """No padding: frame l covers samples [l*hop, l*hop+N) (reading R3)."""
    return 0 if L < N else 1 + (L - N) // hop


def extract_frames(audio: np.ndarray, n_frames: int, M: int, N: int, channel_stride: int,
                   frame_stride: int) -> np.ndarray:
    """Sample n of channel m in frame l is audio.flat[m*channel_stride + l*frame_stride + n] (boundary §(b))."""
    flat = np.asarray(audio).reshape(-1)
    out = np.empty((n_frames, M, N), dtype=np.float64)
    for l in range(n_frames):
        for m in range(M):
            o = m * channel_stride + l * frame_stride
            out[l, m] = flat[o:o + N]
    return out


def sine_window(N: int) -> np.ndarray:
    """w[n] = sin(pi (n + 1/2) / N) ("sine window"; reading R1)."""
    return np.sin(np.pi * (np.arange(N) + 0.5) / N)


def dft_matrix(N: int) -> np.ndarray:
    """(N, N/2+1) matrix of e^{-j 2 pi k n / N}, k = 0..N/2 (sign reading R2)."""
    n = np.arange(N)[:, None]
    k = np.arange(N // 2 + 1)[None, :]
    return np.exp(-2j * np.pi * ((n * k) % N) / N)


def stft(frames: np.ndarray) -> np.ndarray:
    """X^l_m[k] = sum_n w[n] x_m[l*hop + n] e^{-j2pi kn/N} by an explicit DFT matrix.  (F,M,N)->(F,M,K)."""
    N = frames.shape[-1]
    return (frames * sine_window(N)) @ dft_matrix(N)


# ---------------------------------------------------------------- PHAT (eq. 3) and the vector X (eq. 7)
def phat_phasors(X: np.ndarray) -> np.ndarray:
    """X_m[k] / |X_m[k]|, and 0 where |X_m[k]| = 0 (reading R4).  Eq. 3 factorises into these phasors."""
    mag = np.abs(X)
    out = np.zeros_like(X)
    nz = mag > 0
    out[nz] = X[nz] / mag[nz]
    return out


def cross_spectrum(X: np.ndarray) -> np.ndarray:
    """Eq. 3 for every pair, concatenated pair-major with bins inner as eq. 7.

    X_{i,j}[k] = X_i[k] X_j[k]^* / (|X_i[k]| |X_j[k]|), 0 if either magnitude is 0.  (F, M, K) -> (F, P*K).
    """
    F, M, K = X.shape
    out = np.zeros((F, M * (M - 1) // 2, K), dtype=np.complex128)
    for p, (i, j) in enumerate(pairs(M)):
        num = X[:, i, :] * np.conj(X[:, j, :])
        den = np.abs(X[:, i, :]) * np.abs(X[:, j, :])
        nz = den > 0
        out[:, p, :][nz] = num[nz] / den[nz]
    return out.reshape(F, -1)


# ---------------------------------------------------------------- steering matrix W (eqs. 4, 8)
def steering_rows(tau_rows: np.ndarray, N: int) -> np.ndarray:
    """W_{q,i,j}[k] = exp(2 pi sqrt(-1) k tau_{q,i,j} / N) (eq. 4) laid out as eq. 8.

    tau_rows (q, P) -> (q, P*(N/2+1)) complex128.
    """
    k = np.arange(N // 2 + 1, dtype=np.float64)
    ph = 2.0 * np.pi * tau_rows[:, :, None] * k[None, None, :] / N
    return np.exp(1j * ph).reshape(tau_rows.shape[0], -1)


def steering_cols(tau: np.ndarray, N: int, c0: int, c1: int) -> np.ndarray:
    """Columns [c0, c1) of W (all Q rows); column c is pair c // K, bin c % K (eq. 8)."""
    K = N // 2 + 1
    cols = np.arange(c0, c1)
    p, k = cols // K, (cols % K).astype(np.float64)
    return np.exp(1j * 2.0 * np.pi * tau[:, p] * k[None, :] / N)


# ---------------------------------------------------------------- SRP energy and argmax (eqs. 5, 6, 9)
def srp_energy(tau: np.ndarray, x: np.ndarray, N: int, chunk: int = 256) -> np.ndarray:
    """Y = Re{W X} (eq. 9), W generated in row chunks.  x (F, PK) -> Y (F, Q)."""
    Q = tau.shape[0]
    Y = np.empty((x.shape[0], Q))
    for q0 in range(0, Q, chunk):
        W = steering_rows(tau[q0:q0 + chunk], N)
        Y[:, q0:q0 + chunk] = np.real(x @ W.T)
    return Y


def srp_energy_direct(tau_row: np.ndarray, X: np.ndarray, N: int) -> float:
    """Eq. 5 as the literal triple sum for one candidate and one frame.  X (M, K) complex spectra."""
    M, K = X.shape
    tot = 0.0
    for p, (i, j) in enumerate(pairs(M)):
        for k in range(K):
            den = abs(X[i, k]) * abs(X[j, k])
            if den > 0:
                tot += (np.exp(2j * np.pi * k * tau_row[p] / N) * X[i, k] * np.conj(X[j, k]) / den).real
    return tot


def argmax_tie(scores: np.ndarray, rel: float = 1e-9) -> tuple[np.ndarray, np.ndarray]:
    """Eq. 6 per row: lowest index among scores within rel*|best| of the best (readings R10, R11)."""
    best = scores.max(axis=1, keepdims=True)
    ok = scores >= best - rel * np.abs(best)
    q = np.argmax(ok, axis=1)
    return q, scores[np.arange(scores.shape[0]), q]


def degenerate(x: np.ndarray) -> np.ndarray:
    """A frame whose X vector (eq. 7) is identically 0 has no defined argmax (reading R4): q = -1, score 0."""
    return ~np.any(x != 0, axis=1)


def srp_localize(tau: np.ndarray, x: np.ndarray, N: int) -> tuple[np.ndarray, np.ndarray]:
    """SRP-PHAT per frame: q_bar (eq. 6) and Y_q_bar (eq. 5).  Returns (q int64, score float64)."""
    Y = srp_energy(tau, x, N)
    q, s = argmax_tie(Y)
    dg = degenerate(x)
    q[dg] = -1
    s[dg] = 0.0
    return q, s


def frames_to_x(frames: np.ndarray) -> np.ndarray:
    """Alg. 1 online step 1: frames (F, M, N) -> X vector (F, P*K)."""
    return cross_spectrum(stft(frames))


# ---------------------------------------------------------------- multi-source extension (NEXT-1)
def steering_classes(tau: np.ndarray) -> np.ndarray:
    """Representative (lowest) point index of each set of identical steering rows (reading R11), ascending."""
    _, first = np.unique(tau, axis=0, return_index=True)
    return np.sort(first)


def topk_peaks(P: np.ndarray, dirs: np.ndarray, reps: np.ndarray, k: int, sep_deg: float,
               rel: float = 1e-9) -> np.ndarray:
    """The paper names multiple-source localisation as future work without an algorithm; reading R21:
    greedy peaks of the power map P (F, Q) over the steering classes `reps`, each round taking the best class not
    within sep_deg of an earlier peak (unit directions `dirs`, from the array centroid), lowest index among near-ties.
    Returns (F, k) point indices, -1 when no candidate is left."""
    cs = np.cos(np.radians(sep_deg))
    out = -np.ones((P.shape[0], k), dtype=np.int64)
    D = dirs[reps]
    for f in range(P.shape[0]):
        alive = np.ones(len(reps), dtype=bool)
        for j in range(k):
            if not alive.any():
                break
            v = np.where(alive, P[f, reps], -np.inf)
            best = v.max()
            c = int(np.argmax(alive & (v >= best - rel * abs(best))))
            out[f, j] = reps[c]
            alive &= (D @ D[c]) < cs
    return out


def apply_tf_mask(x: np.ndarray, P: int, keep: np.ndarray) -> np.ndarray:
    """Binary time-frequency mask (NEXT-3): X entries (eq. 7) of excluded bins are 0.
    x (F, P*K), keep (F, K) bool -> masked copy of x."""
    F = x.shape[0]
    return (x.reshape(F, P, -1) * keep[:, None, :]).reshape(F, -1)
