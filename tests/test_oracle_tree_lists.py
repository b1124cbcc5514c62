"""Pins for oracle/tree.py and oracle/lists.py.

Structural facts fixed by the definitions (DESIGN.md
readings R3/R4): leaves partition the points, route coverage is exactly once
(brute force over all leaf pairs), and complete uniform grids give closed-form
list totals.
"""
import numpy as np
import pytest

from oracle import lists as L
from oracle.tree import Tree


def _random_tree(seed, n, cap, clustered):
    rng = np.random.default_rng(seed)
    if clustered:
        c = rng.random((3, 3))
        pts = np.concatenate([np.clip(cc + 0.03 * rng.standard_normal((n // 3, 3)), 0, 0.999999) for cc in c])
    else:
        pts = rng.random((n, 3))
    return Tree(pts, cap, max_level=7)


def test_single_root_leaf():
    t = Tree(np.random.default_rng(0).random((1000, 3)), 2000)
    assert t.nbox == 1 and t.leaf[0]
    U, V, W, X = L.all_lists(t)
    assert U[0] == [0] and V[0] == [] and W[0] == [] and X[0] == []


@pytest.mark.parametrize("seed", range(4))
def test_leaves_partition_points_and_respect_cap(seed):
    t = _random_tree(seed, 600, 5, seed % 2 == 1)
    leaves = t.leaves()
    allpts = np.concatenate([t.pts[b] for b in leaves])
    assert np.array_equal(np.sort(allpts), np.arange(600))
    for b in range(t.nbox):
        l = t.level[b]
        # every point of the box has the box's key prefix
        assert np.all((t.q[t.pts[b]] >> (21 - l)) == np.array(t.ijk[b]))
        if t.leaf[b] and l < 7:
            assert t.pts[b].size <= 5
        if not t.leaf[b]:
            assert t.pts[b].size > 5
            kids = [c for c in t.child[b] if c >= 0]
            assert sum(t.pts[c].size for c in kids) == t.pts[b].size
            for o, c in enumerate(t.child[b]):
                if c >= 0:
                    assert t.octant(c) == o and t.parent[c] == b


def _route_counts(t, U, V, W, X):
    """For every (target leaf, source leaf) count the routes that carry the pair."""
    leaves = [int(b) for b in t.leaves()]
    anc = {b: set(t.ancestors(b)) for b in leaves}
    cnt = {}
    for tb in leaves:
        for sb in leaves:
            c = 0
            if sb in U[tb]:
                c += 1
            for ta in anc[tb]:              # M->L at any ancestor pair
                for sa in V[ta]:
                    if sa in anc[sb]:
                        c += 1
            for d in W[tb]:                 # M->T: d is sb or one of its ancestors
                if d in anc[sb]:
                    c += 1
            for ta in anc[tb]:              # S->L: sb in X of tb or an ancestor
                if sb in X[ta]:
                    c += 1
            cnt[(tb, sb)] = c
    return cnt


@pytest.mark.parametrize("seed", range(8))
def test_route_coverage_exactly_once(seed):
    t = _random_tree(seed, 150 + 30 * seed, 3 + seed % 4, seed % 2 == 1)
    U, V, W, X = L.all_lists(t)
    cnt = _route_counts(t, U, V, W, X)
    bad = {k: v for k, v in cnt.items() if v != 1}
    assert not bad, list(bad.items())[:5]
    assert t.depth >= 3


@pytest.mark.parametrize("seed", range(6))
def test_x_list_characterisation_matches_inversion(seed):
    t = _random_tree(100 + seed, 400, 4, seed % 2 == 0)
    _, _, _, X = L.all_lists(t)
    for b in range(t.nbox):
        assert sorted(L.x_list_direct(t, b)) == sorted(X[b])


def _grid_tree(level):
    g = 1 << level
    ax = (np.arange(g) + 0.5) / g
    pts = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), -1).reshape(-1, 3)
    return Tree(pts, 1)


def test_complete_grid_list_totals():
    # complete level-2 grid (4^3 leaves): (3n-2)^3 U pairs, 3096 V pairs, interior |V| = 37
    t = _grid_tree(2)
    assert len(t.leaves()) == 64 and t.depth == 2
    U, V, W, X = L.all_lists(t)
    assert sum(len(U[b]) for b in t.leaves()) == (3 * 4 - 2) ** 3
    assert sum(len(V[b]) for b in t.boxes_at(2)) == 3096
    assert all(len(W[b]) == 0 for b in t.leaves())
    assert all(len(X[b]) == 0 for b in range(t.nbox))
    inner = t.index[(2, 1, 1, 1)]
    assert len(V[inner]) == 64 - 27


def test_complete_level3_grid_v_totals_and_interior_189():
    t = _grid_tree(3)
    V = {b: L.v_list(t, b) for b in t.boxes_at(3)}
    assert sum(len(v) for v in V.values()) == 53352
    b = t.index[(3, 3, 4, 3)]
    assert len(V[b]) == 189
    offs = {tuple(t.ijk_arr[c] - t.ijk_arr[bb]) for bb in V for c in V[bb]}
    assert len(offs) == 316
