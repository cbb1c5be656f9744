"""Parity helpers: run the CUDA path through the C-ABI binding and the float64 oracle on the same seeded input,
and compare them with the north_star rules:

  * framing / indexing bit-exact (the oracle frames the same flat buffer with the same strides itself);
  * DOA indices agree on >= 99.5% of frames, and every disagreement g != o is a near-tie of the oracle's own
    power: P_ref[o] - P_ref[g] <= 2e-3 * |P_ref[o]|  (SRP: Y of eq. 5; SVD: Re{Dhat_q . Zhat}, eq. 14);
  * scores Y_q (eq. 5 at the returned q) within 2e-3 * |Y_ref(q)| of the oracle's Y at that same q.
"""
from __future__ import annotations

import numpy as np

from oracle import srpphat as srp
from oracle import svdphat as svd

TOL = 2e-3
AGREE = 0.995


def oracle_inputs(w, frames_idx=None):
    """Oracle's own framing of the workload buffer (boundary §(b) addressing) -> frames (F, M, N) float64, x."""
    fr = srp.extract_frames(w.audio, w.n_frames, w.M, w.N, w.channel_stride, w.frame_stride) \
        if frames_idx is None else _frames_subset(w, frames_idx)
    return fr, srp.frames_to_x(fr)


def _frames_subset(w, idx):
    flat = w.audio.reshape(-1)
    out = np.empty((len(idx), w.M, w.N))
    for r, l in enumerate(idx):
        for m in range(w.M):
            o = m * w.channel_stride + int(l) * w.frame_stride
            out[r, m] = flat[o:o + w.N]
    return out


def compare(q_gpu, s_gpu, P_ref, Y_at, tag=""):
    """q_gpu/s_gpu: GPU outputs for F frames; P_ref (F, Q): the oracle power used for the argmax;
    Y_at(f, q) -> oracle eq.-5 score of frame f at candidate q.  Returns a dict of stats; raises on violation."""
    F = len(q_gpu)
    q_or, _ = srp.argmax_tie(P_ref)
    agree = q_gpu == q_or
    frac = float(np.mean(agree)) if F else 1.0
    bad = []
    for f in np.nonzero(~agree)[0]:
        g, o = int(q_gpu[f]), int(q_or[f])
        if g < 0 or g >= P_ref.shape[1]:
            bad.append((f, g, o, np.inf))
            continue
        gap = P_ref[f, o] - P_ref[f, g]
        if gap > TOL * abs(P_ref[f, o]):
            bad.append((f, g, o, gap / abs(P_ref[f, o])))
    serr = []
    for f in range(F):
        g = int(q_gpu[f])
        if g >= 0:
            y = Y_at(f, g)
            serr.append(abs(float(s_gpu[f]) - y) / max(abs(y), 1e-30))
    st = dict(frames=F, agree=frac, n_disagree=int(np.sum(~agree)), violations=bad[:10],
              max_score_rel_err=float(max(serr)) if serr else 0.0)
    assert frac >= AGREE, f"{tag}: DOA agreement {frac:.4f} < {AGREE} ({st})"
    assert not bad, f"{tag}: disagreements that are not near-ties: {bad[:10]}"
    assert st["max_score_rel_err"] <= TOL, f"{tag}: score rel err {st['max_score_rel_err']:.2e} > {TOL}"
    return st


def srp_reference(tau, x, N):
    """Oracle SRP powers for all candidates (F, Q) and an eq.-5 scorer."""
    Y = srp.srp_energy(tau, x, N)
    return Y, (lambda f, q: float(Y[f, q]))


def svd_reference(fac, tau, x, N):
    """Oracle SVD-PHAT search powers Re{Dhat_q Zhat} (F, Q) and the eq.-5 scorer from the W row (Alg. 1 step 4)."""
    Z = svd.project(fac["V"], x)
    nz = np.linalg.norm(Z, axis=1, keepdims=True)
    S = svd.search_scores(fac["Rhat"], Z / np.where(nz > 0, nz, 1.0))

    def Y_at(f, q):
        return float(np.real(srp.steering_rows(tau[q:q + 1], N)[0] @ x[f]))
    return S, Y_at
