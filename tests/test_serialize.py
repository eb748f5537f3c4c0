"""Plan-input persistence: save_problem / load_problem round trip (CPU)."""

import dataclasses

import numpy as np

from paper_1801_03589_b200 import geometry as geo
from paper_1801_03589_b200 import load_problem, save_problem
from paper_1801_03589_b200.operators import NesaParams, build_tables
from paper_1801_03589_b200.quadtree import TreeArrays, TreeParams, build_tree


def test_problem_round_trip(tmp_path):
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=2), 20000)
    tree = build_tree(pts, TreeParams(P=48))
    tables = build_tables(tree, NesaParams(Q=16))
    path = str(tmp_path / "c.npz")
    save_problem(path, tree, tables)
    t2, tab2 = load_problem(path)
    for f in dataclasses.fields(TreeArrays):
        a, b = getattr(tree.arrays, f.name), getattr(t2.arrays, f.name)
        if isinstance(a, dict):
            assert a == b
        else:
            assert np.array_equal(a, b) and np.asarray(a).dtype == np.asarray(b).dtype
    assert (t2.l0, t2.L, t2.root_origin, t2.root_side) == (tree.l0, tree.L, tree.root_origin,
                                                        tree.root_side)
    assert np.array_equal(t2.perm, tree.perm) and np.array_equal(t2.points, tree.points)
    assert t2.params == tree.params and tab2.params == tables.params
    for name in ("C", "B", "D", "d_keys", "d_index", "quad", "leaf_center", "leaf_h"):
        assert np.array_equal(getattr(tab2, name), getattr(tables, name))
    for lv in tables.out_fit:
        assert np.array_equal(tab2.out_fit[lv], tables.out_fit[lv])
        assert np.array_equal(tab2.in_fit[lv], tables.in_fit[lv])
    # the tree alone
    save_problem(str(tmp_path / "t.npz"), tree)
    t3, none = load_problem(str(tmp_path / "t.npz"))
    assert none is None and np.array_equal(t3.arrays.int_idx, tree.arrays.int_idx)
