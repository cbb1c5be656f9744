"""Exact k-d tree nearest-neighbour search (Alg. 1 offline 4 / online 3).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The paper names only "a k-d tree" (Bentley 1975); this is
the textbook exact construction: split at the median of the coordinate with the widest spread, leaves of <= 16
points scanned exhaustively, branch-and-bound search that visits a far child unless its splitting plane is
strictly farther than the current best.  Ties are broken by the lowest point index (reading R10), so the
result equals the brute-force scan exactly.
"""
from __future__ import annotations

import numpy as np


class KDTree:
    def __init__(self, points: np.ndarray, leaf_size: int = 16):
        self.pts = np.asarray(points, dtype=np.float64)
        if self.pts.ndim != 2 or self.pts.shape[0] == 0:
            raise ValueError("k-d tree needs a non-empty (n, dim) point set")
        self.leaf = leaf_size
        # node arrays: for internal nodes dim >= 0, leaves dim = -1 and [lo, hi) into self.order
        self.dim, self.val, self.left, self.right, self.lo, self.hi = [], [], [], [], [], []
        self.order = np.arange(self.pts.shape[0])
        self.visited = 0
        self._build(0, self.pts.shape[0])

    def _new(self) -> int:
        for a in (self.dim, self.val, self.left, self.right, self.lo, self.hi):
            a.append(0)
        return len(self.dim) - 1

    def _build(self, lo: int, hi: int) -> int:
        n = self._new()
        idx = self.order[lo:hi]
        self.lo[n], self.hi[n] = lo, hi
        if hi - lo <= self.leaf:
            self.dim[n] = -1
            return n
        sub = self.pts[idx]
        spread = sub.max(axis=0) - sub.min(axis=0)
        d = int(np.argmax(spread))
        if spread[d] == 0.0:                       # all points identical: leaf
            self.dim[n] = -1
            return n
        srt = idx[np.argsort(sub[:, d], kind="stable")].copy()
        self.order[lo:hi] = srt
        mid = lo + (hi - lo) // 2
        self.dim[n], self.val[n] = d, float(self.pts[srt[mid - lo], d])
        # left: [lo, mid) (coords <= val), right: [mid, hi) (coords >= val)
        self.left[n] = self._build(lo, mid)
        self.right[n] = self._build(mid, hi)
        return n

    def nearest(self, q: np.ndarray) -> tuple[int, float]:
        """Exact argmin_i ||p_i - q||^2, ties -> lowest i.  Returns (index, squared distance)."""
        best = [np.inf, -1]
        self._search(0, np.asarray(q, dtype=np.float64), best)
        return int(best[1]), float(best[0])

    def _search(self, n: int, q: np.ndarray, best: list) -> None:
        self.visited += 1
        if self.dim[n] < 0:
            for i in self.order[self.lo[n]:self.hi[n]]:
                diff = self.pts[i] - q
                d2 = float(diff @ diff)
                if d2 < best[0] or (d2 == best[0] and i < best[1]):
                    best[0], best[1] = d2, int(i)
            return
        d, v = self.dim[n], self.val[n]
        near, far = (self.left[n], self.right[n]) if q[d] <= v else (self.right[n], self.left[n])
        self._search(near, q, best)
        gap = q[d] - v
        if gap * gap <= best[0]:                   # equal distance may still hold a lower index: visit
            self._search(far, q, best)

    def within(self, q: np.ndarray, r2: float) -> list[int]:
        """All point indices with squared distance <= r2."""
        out: list[int] = []
        self._range(0, np.asarray(q, dtype=np.float64), r2, out)
        return out

    def _range(self, n: int, q: np.ndarray, r2: float, out: list) -> None:
        if self.dim[n] < 0:
            for i in self.order[self.lo[n]:self.hi[n]]:
                diff = self.pts[i] - q
                if float(diff @ diff) <= r2:
                    out.append(int(i))
            return
        d, v = self.dim[n], self.val[n]
        gap = q[d] - v
        if gap <= 0 or gap * gap <= r2:
            self._range(self.left[n], q, r2, out)
        if gap >= 0 or gap * gap <= r2:
            self._range(self.right[n], q, r2, out)

    def nearest_tie(self, q: np.ndarray, tol: float = 1e-9) -> int:
        """Lowest index among points within tol (squared distance) of the nearest (readings R10/R11)."""
        _, d2 = self.nearest(q)
        return min(self.within(q, d2 + tol))
