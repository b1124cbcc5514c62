"""Adaptive octree by midpoint recursion (oracle; test infrastructure).

Definition followed (readings R4):
  * root box = [0,1)^3 (level 0);
  * quantise q = floor(x * 2^21), clamped to [0, 2^21 - 1];
  * box (l; i,j,k) has half-width h_l = 2^-(l+1) and centre ((i,j,k) + 1/2) / 2^l;
  * a box splits iff its point count > cap and l < 20 ("no more
    than 2000 target points" with the BASELINE cap in place of 2000);
  * a split distributes the box's points to the 8 children by comparing each
    quantised coordinate with the box's integer midpoint; only non-empty
    children are kept (an empty child carries no work);
  * no 2:1 balancing.
The paper describes the octree only as "spatial adaptive octree"
(PAPER.md:14, :53); the rest is the standard KIFMM construction.
"""
from __future__ import annotations

import numpy as np

QBITS = 21
MAX_LEVEL = 20


class Tree:
    """Plain list-of-boxes octree.

    box b: level[b], ijk[b] (3 ints at its level), parent[b] (-1 for root),
    child[b][oct] (box id or -1; oct = 4*cx + 2*cy + cz), leaf[b],
    pts[b] = original point indices inside the box (ascending).
    Boxes are stored level by level (BFS order).
    """

    def __init__(self, points: np.ndarray, cap: int, max_level: int = MAX_LEVEL):
        points = np.asarray(points, dtype=np.float64)
        n = points.shape[0]
        q = np.floor(points * float(1 << QBITS)).astype(np.int64)
        q = np.clip(q, 0, (1 << QBITS) - 1)
        self.q = q
        self.n = n
        self.cap = cap
        self.level: list[int] = []
        self.ijk: list[tuple] = []
        self.parent: list[int] = []
        self.child: list[list[int]] = []
        self.leaf: list[bool] = []
        self.pts: list[np.ndarray] = []
        self._new(0, (0, 0, 0), -1, np.arange(n, dtype=np.int64))
        b = 0
        while b < len(self.level):
            l = self.level[b]
            idx = self.pts[b]
            if idx.size > cap and l < max_level:
                self.leaf[b] = False
                shift = QBITS - 1 - l  # bit selecting the child half at level l+1
                i, j, k = self.ijk[b]
                cx = (q[idx, 0] >> shift) & 1
                cy = (q[idx, 1] >> shift) & 1
                cz = (q[idx, 2] >> shift) & 1
                octant = 4 * cx + 2 * cy + cz
                for o in range(8):
                    sel = idx[octant == o]
                    if sel.size == 0:
                        continue
                    ox, oy, oz = (o >> 2) & 1, (o >> 1) & 1, o & 1
                    c = self._new(l + 1, (2 * i + ox, 2 * j + oy, 2 * k + oz), b, sel)
                    self.child[b][o] = c
            b += 1
        self.nbox = len(self.level)
        self.level_arr = np.array(self.level, dtype=np.int64)
        self.ijk_arr = np.array(self.ijk, dtype=np.int64).reshape(-1, 3)
        self.leaf_arr = np.array(self.leaf, dtype=bool)
        self.depth = int(self.level_arr.max())
        self.index = {(self.level[b],) + tuple(self.ijk[b]): b for b in range(self.nbox)}
        # integer extents in units of the finest quantum (closed boxes)
        sh = QBITS - self.level_arr
        self.lo = self.ijk_arr << sh[:, None]
        self.hi = (self.ijk_arr + 1) << sh[:, None]

    def _new(self, level, ijk, parent, pts):
        self.level.append(level)
        self.ijk.append(tuple(int(v) for v in ijk))
        self.parent.append(parent)
        self.child.append([-1] * 8)
        self.leaf.append(True)
        self.pts.append(pts)
        return len(self.level) - 1

    # geometry
    def centre(self, b: int) -> np.ndarray:
        return (np.array(self.ijk[b], dtype=np.float64) + 0.5) / float(1 << self.level[b])

    def half_width(self, b: int) -> float:
        return 0.5 / float(1 << self.level[b])

    def octant(self, b: int) -> int:
        i, j, k = self.ijk[b]
        return 4 * (i & 1) + 2 * (j & 1) + (k & 1)

    def leaves(self) -> np.ndarray:
        return np.nonzero(self.leaf_arr)[0]

    def boxes_at(self, l: int) -> np.ndarray:
        return np.nonzero(self.level_arr == l)[0]

    def adjacent(self, a: int, b: int) -> bool:
        """Closed boxes intersect."""
        return bool(np.all(self.lo[a] <= self.hi[b]) and np.all(self.lo[b] <= self.hi[a]))

    def adjacent_many(self, a: int, bs: np.ndarray) -> np.ndarray:
        return np.all(self.lo[a] <= self.hi[bs], axis=1) & np.all(self.lo[bs] <= self.hi[a], axis=1)

    def ancestors(self, b: int) -> list[int]:
        out = []
        while b >= 0:
            out.append(b)
            b = self.parent[b]
        return out
