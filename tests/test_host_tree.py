"""Bit-exact pins of the host tree build against the reference's own output.

Fixtures in tests/golden were produced by oracle/gen_golden.py running the
reference (taskfmm.quadtree.build_tree, quadtree.py:123-245).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, GOLDEN_CASES, grid_points, have_reference
from paper_1801_03589_b200 import geometry as geo
from paper_1801_03589_b200.quadtree import TreeParams, build_tree, tree_stats


def tree_arrays(tree):
    from oracle.gen_golden import tree_arrays as ta
    return ta(tree)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_tree_matches_reference(golden, name):
    g = golden(name)
    tree = build_tree(g["points"], TreeParams(P=int(g["P"])))
    mine = tree_arrays(tree)
    from oracle.gen_golden import tree_digest
    assert tree_digest(mine) == str(g["tree_sha256"])
    for k, v in mine.items():
        if f"tree_{k}" in g:
            assert np.array_equal(v, g[f"tree_{k}"]), k


def _digest_rows():
    rows = {}
    with open(os.path.join(GOLDEN, "tree_digests.txt")) as f:
        for line in f:
            name, dig, L, G = line.split()
            rows[name] = (dig, int(L), int(G))
    return rows


@pytest.mark.parametrize("name,spec,n,P", [
    ("wave_200000_P48", geo.CurveSpec(), 200000, 48),
    ("ellipse_plates_200000_P48", geo.CurveSpec(kind="ellipse-plates", seed=2), 200000, 48),
    ("circle_random_20000_P32", geo.CurveSpec(kind="circle-random", seed=1), 20000, 32),
])
def test_tree_digest_large(name, spec, n, P):
    from oracle.gen_golden import tree_digest
    dig, L, G = _digest_rows()[name]
    tree = build_tree(geo.generate_sources(spec, n), TreeParams(P=P))
    assert tree.L == L and tree.arrays.n_groups == G
    assert tree_digest(tree_arrays(tree)) == dig


@pytest.mark.slow
def test_tree_digest_c4_2m():
    from oracle.gen_golden import tree_digest
    dig, L, G = _digest_rows()["ellipse_plates_2000000_P64"]
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=3), 2000000)
    tree = build_tree(pts, TreeParams(P=64))
    assert (tree.L, tree.arrays.n_groups) == (L, G)
    assert tree_digest(tree_arrays(tree)) == dig


def test_grid_stopping_rule_and_lists():
    # quadtree tests of the reference (test_quadtree.py:14-112) restated
    tree = build_tree(grid_points(4), TreeParams(P=1))
    assert tree.l0 == 2 and tree.L == 2 and len(tree.leaves()) == 16
    tree = build_tree(grid_points(16), TreeParams(P=1))
    assert tree.L == 4
    by = {(g.ix, g.iy): g for g in tree.leaves()}
    assert len(by[(7, 7)].neighbors) == 9 and len(by[(0, 0)].neighbors) == 4
    coarse = [tree.groups[i] for i in tree.level_ids[2]]
    assert all(len(g.interaction) <= 12 for g in coarse)
    st = tree_stats(tree)
    for lv in range(tree.l0, tree.L):
        assert st["groups_per_level"][lv + 1] == 4 * st["groups_per_level"][lv]


def test_build_rejections():
    with pytest.raises(ValueError):
        build_tree(np.array([[0.0, 0.0], [1.0, 1.0], [0.0, 0.0], [2.0, 0.0]]), TreeParams())
    with pytest.raises(ValueError):
        build_tree(np.array([[0.0, 0.0], [1.0, 1.0]]), TreeParams())
    with pytest.raises(ValueError):
        TreeParams(P=0)
    with pytest.raises(ValueError):
        TreeParams(l0_groups_longest=3)


def test_near_far_cover_once():
    # every leaf pair is near or far at exactly one level (test_quadtree.py:129-156)
    tree = build_tree(geo.generate_sources(geo.CurveSpec(), 1000), TreeParams(P=10))
    leaves = tree.leaves()
    anc = {}
    for g in leaves:
        chain, cur = {}, g
        while True:
            chain[cur.level] = cur.id
            if cur.parent is None:
                break
            cur = tree.groups[cur.parent]
        anc[g.id] = chain
    inter = [set(g.interaction) for g in tree.groups]
    for a in leaves:
        nb = set(a.neighbors)
        for b in leaves:
            far = sum(anc[b.id][lv] in inter[anc[a.id][lv]] for lv in range(tree.l0, tree.L + 1))
            assert (b.id in nb) + far == 1


@pytest.mark.skipif(not have_reference(), reason="reference not mounted (GPU box)")
def test_reference_tree_adapter_roundtrip():
    import sys
    from conftest import REFERENCE_SRC
    sys.path.insert(0, REFERENCE_SRC)
    from taskfmm import quadtree as RQ
    from paper_1801_03589_b200.fastmvp import as_tree
    pts = geo.generate_sources(geo.CurveSpec(kind="annulus-random", seed=4), 3000)
    rt = RQ.build_tree(pts, RQ.TreeParams(P=20))
    a = as_tree(rt).arrays
    b = build_tree(pts, TreeParams(P=20)).arrays
    for f in ("level", "ix", "iy", "start", "stop", "parent", "child_first", "n_children",
              "box", "nbr_ptr", "nbr_idx", "int_ptr", "int_idx"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("spec,n,P", [
    (geo.CurveSpec(), 1500, 40),
    (geo.CurveSpec(kind="circle-random", seed=1), 20000, 32),
    (geo.CurveSpec(kind="ellipse-plates", seed=2), 200000, 48),
    (geo.CurveSpec(kind="circle", seed=3), 5000, 20),
])
def test_native_tree_build_bit_identical_to_numpy(spec, n, P):
    # csrc/nesa_tree.cpp (the C++ build, default) against the numpy restatement
    from oracle.gen_golden import tree_arrays as ta
    pts = geo.generate_sources(spec, n)
    a = build_tree(pts, TreeParams(P=P), native=True)
    b = build_tree(pts, TreeParams(P=P), native=False)
    A, B = ta(a), ta(b)
    assert set(A) == set(B)
    for k in B:
        assert np.array_equal(A[k], B[k]), k
    assert (a.l0, a.L, a.root_side, a.root_origin) == (b.l0, b.L, b.root_side, b.root_origin)
    assert np.array_equal(a.points, b.points)


@pytest.mark.parametrize("native", [True, False])
def test_tree_build_errors(native):
    pts = geo.generate_sources(geo.CurveSpec(), 500)
    dup = pts.copy()
    dup[3] = dup[100]
    with pytest.raises(ValueError, match="distinct"):
        build_tree(dup, TreeParams(P=20), native=native)
    with pytest.raises(ValueError):
        build_tree(pts[:3], TreeParams(P=2, l0_groups_longest=4), native=native)
    same = np.zeros((4, 2))
    with pytest.raises(ValueError):
        build_tree(same, TreeParams(P=1), native=native)
