"""Array geometries and candidate grids for the five BASELINE.json configs and the paper's Tables 1-2.

This module builds INPUTS only (microphone positions, candidate directions/points).  It holds none of the
method's arithmetic (no TDOA, no steering, no STFT); both the oracle (`oracle/`) and the CUDA path consume
its outputs.

Citations: PAPER.md line numbers (`P:n`) and BASELINE.json configs (`BJ.cfgN`, 1-based).
"""
from __future__ import annotations

import numpy as np

FS = 16000.0          # P:218 Table 1; BJ.cfg1-5
C_SOUND = 343.0       # P:218 Table 1; BJ.cfg1


# --------------------------------------------------------------------------------------------------------------
# Candidate DOA grid: "equidistant points on a unit sphere generated recursively ... for a total of 2562 points"
# (P:208).  2562 = 10*4^4+2 is the vertex count of an icosahedron subdivided 4 times (SPEC S:73 decision;
# DESIGN.md reading R5).  Level 5 gives the 10242 points of BJ.cfg3/cfg4.
# --------------------------------------------------------------------------------------------------------------
def icosphere(level: int) -> np.ndarray:
    """Vertices (Q x 3, float64, unit norm) of an icosahedron whose faces are split 4-way `level` times.

    Order: the 12 base vertices, then midpoints in creation order.  The construction is exactly symmetric
    under z -> -z (mirrored vertices have bitwise-identical x, y and negated z), which is what makes the
    twin rows of planar arrays bitwise identical (reading R11).
    """
    if level < 0 or level > 8:
        raise ValueError("icosphere level must be in [0, 8]")
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    base = [(-1, phi, 0), (1, phi, 0), (-1, -phi, 0), (1, -phi, 0),
            (0, -1, phi), (0, 1, phi), (0, -1, -phi), (0, 1, -phi),
            (phi, 0, -1), (phi, 0, 1), (-phi, 0, -1), (-phi, 0, 1)]
    verts = [_unit(np.array(v, dtype=np.float64)) for v in base]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
             (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
             (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
             (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(level):
        cache: dict[tuple[int, int], int] = {}

        def mid(a: int, b: int) -> int:
            key = (a, b) if a < b else (b, a)
            if key not in cache:
                m = (verts[key[0]] + verts[key[1]]) * 0.5
                verts.append(_unit(m))
                cache[key] = len(verts) - 1
            return cache[key]

        new_faces = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            new_faces += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = new_faces
    return np.ascontiguousarray(np.stack(verts))


def _unit(v: np.ndarray) -> np.ndarray:
    n = np.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])
    return v / n


# --------------------------------------------------------------------------------------------------------------
# Paper Table 2: 7-mic 1-D / 2-D / 3-D arrays, positions in cm.
# --------------------------------------------------------------------------------------------------------------
PAPER_TABLE2_CM = {
    "1d": [(0, 0, -5.0), (0, 0, -3.3), (0, 0, -1.7), (0, 0, 0), (0, 0, 1.7), (0, 0, 3.3), (0, 0, 5.0)],
    "2d": [(0, 0, 0), (5, 0, 0), (2.5, 4.3, 0), (-2.5, 4.3, 0), (-5.0, 0, 0), (-2.5, -4.3, 0), (2.5, -4.3, 0)],
    "3d": [(0, 0, 0), (-5, 0, 0), (5, 0, 0), (0, -5, 0), (0, 5, 0), (0, 0, -5), (0, 0, 5)],
}


def paper_array(name: str) -> np.ndarray:
    """Table 2 positions converted to metres."""
    return np.asarray(PAPER_TABLE2_CM[name], dtype=np.float64) / 100.0


# --------------------------------------------------------------------------------------------------------------
# BASELINE.json arrays (readings R15/R16 of DESIGN.md for orientation/order).
# --------------------------------------------------------------------------------------------------------------
def square_array(side: float = 0.1) -> np.ndarray:
    """BJ.cfg1: planar square, z=0, counter-clockwise from (+,+)."""
    h = side / 2.0
    return np.array([(h, h, 0.0), (-h, h, 0.0), (-h, -h, 0.0), (h, -h, 0.0)], dtype=np.float64)


def uca(n: int, radius: float, z: float = 0.0) -> np.ndarray:
    """Uniform circular array, mic m at azimuth 2*pi*m/n (BJ.cfg2)."""
    a = 2.0 * np.pi * np.arange(n) / n
    return np.stack([radius * np.cos(a), radius * np.sin(a), np.full(n, z)], axis=1)


def two_ring_array() -> np.ndarray:
    """BJ.cfg3: rings of 8 at r=0.05 m (z=0; mics 0-7) and r=0.1 m (z=0.05; mics 8-15), aligned azimuths."""
    return np.concatenate([uca(8, 0.05, 0.0), uca(8, 0.10, 0.05)], axis=0)


def random_cube_array(rng: np.random.Generator, n: int = 32, side: float = 0.3) -> np.ndarray:
    """BJ.cfg4: n mics uniform in a side^3 cube centred on the origin, drawn from the config seed."""
    return rng.uniform(-side / 2.0, side / 2.0, size=(n, 3))


def box_grid(mics: np.ndarray) -> np.ndarray:
    """BJ.cfg5 near-field candidate points: 20x20x10 cell-centred lattice (0.1 m pitch) over a 2x2x1 m box whose
    centre is the array centroid + 1.5 m along z (reading R15).  Index q = (ix*20 + iy)*10 + iz."""
    c = mics.mean(axis=0)
    xs = -0.95 + 0.1 * np.arange(20)
    zs = 1.05 + 0.1 * np.arange(10)
    pts = np.empty((4000, 3), dtype=np.float64)
    q = 0
    for ix in range(20):
        for iy in range(20):
            for iz in range(10):
                pts[q] = (c[0] + xs[ix], c[1] + xs[iy], c[2] + zs[iz])
                q += 1
    return pts
