"""U/V/W/X interaction lists by their definitions (oracle; test infrastructure).

The paper names the lists and defines U and V in words (PAPER.md:152-156:
"U-list refers to the octree boxes adjacent to B ... V-list refers to the set
of the children of the neighbors of the parent of B which are not adjacent to
B") and defers W/X to the KIFMM literature ("we omit those technical
details").  Reading R3 pins the standard definitions:

  adjacent(A, B)  the closed boxes intersect;
  colleagues(B)   same-level boxes adjacent to B, B excluded;
  U(B), B leaf    all leaves adjacent to B, B included;
  V(B), any box   children of colleagues of parent(B) not adjacent to B;
  W(B), B leaf    descendants D of B's colleagues with D not adjacent to B
                  and parent(D) adjacent to B;
  X(B), any box   leaves A with B in W(A).
"""
from __future__ import annotations

import numpy as np

from .tree import Tree


def colleagues(t: Tree, b: int) -> list[int]:
    l = t.level[b]
    i, j, k = t.ijk[b]
    out = []
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                if dx == dy == dz == 0:
                    continue
                c = t.index.get((l, i + dx, j + dy, k + dz))
                if c is not None:
                    out.append(c)
    return out


def u_list(t: Tree, b: int) -> list[int]:
    leaves = t.leaves()
    adj = t.adjacent_many(b, leaves)
    return [int(a) for a in leaves[adj]]


def v_list(t: Tree, b: int) -> list[int]:
    if t.parent[b] < 0:
        return []
    out = []
    for c in colleagues(t, t.parent[b]):
        for d in t.child[c]:
            if d >= 0 and not t.adjacent(d, b):
                out.append(d)
    return out


def w_list(t: Tree, b: int) -> list[int]:
    out = []

    def descend(c):
        for d in t.child[c]:
            if d < 0:
                continue
            if not t.adjacent(d, b):
                out.append(d)          # parent c is adjacent to b by construction
            elif not t.leaf[d]:
                descend(d)

    for c in colleagues(t, b):
        if not t.leaf[c]:
            descend(c)
    return out


def x_lists_by_inversion(t: Tree, w: dict) -> dict:
    """X(B) = {A leaf : B in W(A)}, computed literally by inverting the W lists."""
    x: dict = {b: [] for b in range(t.nbox)}
    for a, ws in w.items():
        for b in ws:
            x[b].append(a)
    return x


def x_list_direct(t: Tree, b: int) -> list[int]:
    """X(B) for one box without inverting every W list.

    Equivalent characterisation (lists): A in X(B) iff A is a leaf
    with level(A) < level(B), B not adjacent to A and parent(B) adjacent to A
    -- then the ancestor of B at A's level is a colleague of A and the descent
    of w_list reaches B.  tests/test_oracle_lists.py checks it against
    x_lists_by_inversion on random adaptive trees.
    """
    p = t.parent[b]
    if p < 0:
        return []
    leaves = t.leaves()
    cand = leaves[t.level_arr[leaves] < t.level[b]]
    ok = t.adjacent_many(p, cand) & ~t.adjacent_many(b, cand)
    return [int(a) for a in cand[ok]]


def all_lists(t: Tree):
    """U, W for every leaf; V for every box; X by inverting W."""
    leaves = [int(b) for b in t.leaves()]
    U = {b: u_list(t, b) for b in leaves}
    W = {b: w_list(t, b) for b in leaves}
    V = {b: v_list(t, b) for b in range(t.nbox)}
    X = x_lists_by_inversion(t, W)
    return U, V, W, X
