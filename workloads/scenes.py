"""Seeded synthetic scenes standing in for the paper's TIMIT + image-method data (not available).

Free-field physics only: a white-Gaussian source is delayed per microphone by a fractional delay applied in the
frequency domain, plus independent white Gaussian noise per mic.  Nothing here computes any step of the
localisation method (no TDOA tables, no steering matrix, no STFT, no PHAT).  The recipe is stated in
DESIGN.md ("Input recipe") and follows SURVEY.md §8(d):

  * seed: numpy.random.default_rng(181111785 + cfg)          (cfg is 1-based)
  * plane wave from unit direction u: mic m is delayed by  -(fs/c) r_m . u  samples
  * point source at s: mic m is delayed by (fs/c)||s - r_m|| samples and scaled by 1/||s - r_m||
  * SNR is measured against the mean over mics of the clean signal power (reading R20)
"""
from __future__ import annotations

import numpy as np

PAD = 256  # zero-phase padding (samples) on each side of a segment before the spectral delay


def _random_unit(rng: np.random.Generator, n: int | None = None) -> np.ndarray:
    v = rng.standard_normal((3,) if n is None else (n, 3))
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def delayed_copies(src: np.ndarray, delays: np.ndarray, gains: np.ndarray | None = None) -> np.ndarray:
    """Fractionally delay `src` (..., Lp) by `delays` (..., M) samples -> (..., M, Lp - 2*PAD).

    x_m(t) = g_m * s(t - delay_m), realised as a linear phase ramp on the rfft of the padded segment.
    """
    lp = src.shape[-1]
    spec = np.fft.rfft(src, axis=-1)                                 # (..., Lp/2+1)
    f = np.arange(spec.shape[-1], dtype=np.float64)
    ramp = np.exp(-2j * np.pi * delays[..., :, None] * f / lp)     # (..., M, Lp/2+1)
    out = np.fft.irfft(spec[..., None, :] * ramp, n=lp, axis=-1)[..., PAD:lp - PAD]
    if gains is not None:
        out = out * gains[..., :, None]
    return out


def add_noise(rng: np.random.Generator, clean: np.ndarray, snr_db) -> np.ndarray:
    """White Gaussian noise per mic; SNR vs the mean over mics of the clean power (per leading index)."""
    p_sig = np.mean(clean ** 2, axis=(-2, -1), keepdims=True)
    snr = np.asarray(snr_db, dtype=np.float64)
    snr = snr.reshape(snr.shape + (1,) * (clean.ndim - snr.ndim)) if snr.ndim else snr
    sigma = np.sqrt(p_sig / 10.0 ** (snr / 10.0))
    return clean + sigma * rng.standard_normal(clean.shape)


def plane_wave_delays(mics: np.ndarray, u: np.ndarray, fs: float, c: float) -> np.ndarray:
    """Propagation delay (samples) of a plane wave arriving from unit direction u (..., 3) at each mic."""
    return -(fs / c) * (u @ mics.T)


def plane_wave_stream(rng, mics, fs, c, L, u, snr_db) -> np.ndarray:
    """One plane wave from u over L samples + noise -> (M, L) float64."""
    src = rng.standard_normal(L + 2 * PAD)
    clean = delayed_copies(src, plane_wave_delays(mics, u, fs, c))
    return add_noise(rng, clean, snr_db)


def plane_wave_frames(rng, mics, fs, c, N, dirs, snr_db, dirs2=None, level2_db=None, batch=512):
    """Independent N-sample frames, one (or two) plane waves each -> (B, M, N) float32."""
    B = dirs.shape[0]
    out = np.empty((B, mics.shape[0], N), dtype=np.float32)
    for b0 in range(0, B, batch):
        b1 = min(B, b0 + batch)
        n = b1 - b0
        clean = delayed_copies(rng.standard_normal((n, N + 2 * PAD)), plane_wave_delays(mics, dirs[b0:b1], fs, c))
        if dirs2 is not None:
            g2 = 10.0 ** (-level2_db[b0:b1] / 20.0)
            clean2 = delayed_copies(rng.standard_normal((n, N + 2 * PAD)),
                                    plane_wave_delays(mics, dirs2[b0:b1], fs, c))
            clean = clean + g2[:, None, None] * clean2
        snr = snr_db if np.ndim(snr_db) == 0 else snr_db[b0:b1]
        out[b0:b1] = add_noise(rng, clean, snr).astype(np.float32)
    return out


def point_source_stream(rng, mics, fs, c, L, pos, snr_db) -> np.ndarray:
    d = np.linalg.norm(pos[None, :] - mics, axis=1)
    src = rng.standard_normal(L + 2 * PAD)
    clean = delayed_copies(src, (fs / c) * d, 1.0 / d)
    return add_noise(rng, clean, snr_db)


def frame_count(L: int, N: int, hop: int) -> int:
    """Frames of a stream without padding: 1 + floor((L - N) / hop), 0 if L < N (reading R3)."""
    return 0 if L < N else 1 + (L - N) // hop
