"""The five BASELINE.json configurations (BJ.cfg1..cfg5, 1-based) as seeded synthetic workloads.

`make(cfg, frames=None)` returns a `Workload`: the plan parameters (mics, fs, c, N, hop, field, points, delta)
plus float32 audio in the layout the config names and the ground truth used by injection/sanity tests.
`frames` shrinks a config (same geometry and grid, fewer frames) for oracle-sized parity tests.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import geometry as G
from . import scenes as S

SEED_BASE = 181111785
DEFAULT_FRAMES = {1: 124, 2: 3749, 3: 10_000, 4: 10_000, 5: 100_000}
DELTA = 1e-5  # BJ.cfg1: "keeping 1-1e-5 of the singular-value energy"


@dataclass
class Workload:
    cfg: int
    name: str
    mics: np.ndarray            # (M, 3) metres
    fs: float
    c: float
    N: int
    hop: int
    field: str                  # "far" (eq. 2) or "near" (eq. 1)
    points: np.ndarray          # (Q, 3): unit directions (far) or positions in metres (near)
    delta: float
    audio: np.ndarray           # float32, (M, L) stream or (B, M, N) framed
    layout: str                 # "stream" | "framed"
    n_frames: int
    channel_stride: int         # sample n of channel m in frame l: audio.flat[m*cs + l*fs_ + n]
    frame_stride: int
    frames_per_call: int        # frames per localize call (cfg5: 256)
    truth: dict = field(default_factory=dict)

    @property
    def M(self) -> int:
        return self.mics.shape[0]

    @property
    def Q(self) -> int:
        return self.points.shape[0]


def make(cfg: int, frames: int | None = None) -> Workload:
    if cfg not in DEFAULT_FRAMES:
        raise ValueError("cfg must be 1..5")
    F = DEFAULT_FRAMES[cfg] if frames is None else int(frames)
    rng = np.random.default_rng(SEED_BASE + cfg)
    fs, c = G.FS, G.C_SOUND
    if cfg == 1:
        mics, N, hop = G.square_array(0.1), 512, 256
        L = (F - 1) * hop + N if frames is not None else 32000
        u = S._random_unit(rng)
        audio = S.plane_wave_stream(rng, mics, fs, c, L, u, 5.0).astype(np.float32)
        return _stream(cfg, "square4_far", mics, N, hop, "far", G.icosphere(4), audio, 124 if frames is None else F,
                       {"u": u})
    if cfg == 2:
        mics, N, hop = G.uca(8, 0.05), 512, 256
        L = (F - 1) * hop + N if frames is not None else 960000
        seg, parts, us, snrs = 16000, [], [], []
        for s0 in range(0, L, seg):
            n = min(seg, L - s0)
            u, snr = S._random_unit(rng), rng.uniform(0.0, 20.0)
            parts.append(S.plane_wave_stream(rng, mics, fs, c, n, u, snr))
            us.append(u)
            snrs.append(snr)
        audio = np.concatenate(parts, axis=1).astype(np.float32)
        return _stream(cfg, "uca8_far", mics, N, hop, "far", G.icosphere(4), audio, S.frame_count(L, N, hop),
                       {"u": np.array(us), "snr": np.array(snrs), "segment": seg})
    if cfg == 3:
        mics, N, hop = G.two_ring_array(), 1024, 512
        dirs = S._random_unit(rng, F)
        audio = S.plane_wave_frames(rng, mics, fs, c, N, dirs, 10.0)
        return _framed(cfg, "tworing16_far", mics, N, hop, "far", G.icosphere(5), audio, {"u": dirs})
    if cfg == 4:
        mics = G.random_cube_array(rng, 32, 0.3)
        N, hop = 1024, 512
        d1, d2 = S._random_unit(rng, F), S._random_unit(rng, F)
        lvl = rng.uniform(0.0, 6.0, size=F)
        audio = S.plane_wave_frames(rng, mics, fs, c, N, d1, 5.0, dirs2=d2, level2_db=lvl)
        return _framed(cfg, "cube32_far", mics, N, hop, "far", G.icosphere(5), audio, {"u": d1, "u2": d2,
                                                                                        "level2_db": lvl})
    # cfg == 5: near field, cfg3's 16-mic array (reading R14), 20x20x10 box grid, 256 frames per call
    mics, N, hop = G.two_ring_array(), 512, 256
    pts = G.box_grid(mics)
    L = (F - 1) * hop + N
    seg, parts, pos = 16000, [], []
    ctr = mics.mean(axis=0)
    for s0 in range(0, L, seg):
        n = min(seg, L - s0)
        p = ctr + np.array([rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(1.0, 2.0)])
        parts.append(S.point_source_stream(rng, mics, fs, c, n, p, 10.0))
        pos.append(p)
    audio = np.concatenate(parts, axis=1).astype(np.float32)
    w = _stream(cfg, "tworing16_near", mics, N, hop, "near", pts, audio, F, {"pos": np.array(pos), "segment": seg})
    w.frames_per_call = 256
    return w


def _stream(cfg, name, mics, N, hop, fld, pts, audio, F, truth) -> Workload:
    L = audio.shape[1]
    assert S.frame_count(L, N, hop) == F
    return Workload(cfg, name, mics, G.FS, G.C_SOUND, N, hop, fld, pts, DELTA, audio, "stream", F,
                    channel_stride=L, frame_stride=hop, frames_per_call=F, truth=truth)


def _framed(cfg, name, mics, N, hop, fld, pts, audio, truth) -> Workload:
    B, M, _ = audio.shape
    return Workload(cfg, name, mics, G.FS, G.C_SOUND, N, hop, fld, pts, DELTA, audio, "framed", B,
                    channel_stride=N, frame_stride=M * N, frames_per_call=B, truth=truth)


def frame_view(w: Workload) -> np.ndarray:
    """(F, M, N) float32 view/copy of the workload's frames, addressed exactly as the C-ABI addresses them."""
    if w.layout == "framed":
        return w.audio
    idx = np.arange(w.n_frames)[:, None] * w.hop + np.arange(w.N)[None, :]
    return np.ascontiguousarray(w.audio[:, idx].transpose(1, 0, 2))
