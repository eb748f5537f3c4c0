"""Generate tests/golden/*.npz by running the REFERENCE itself.

Run in the build container (needs /root/reference, read-only):

    python oracle/gen_golden.py          # the small cases + tree digests
    python oracle/gen_golden.py c3       # BASELINE C3 (200k points), phi only

For each case the reference's own ``build_tree`` / ``build_all`` /
``mvp_serial`` / ``dense_matvec`` (taskfmm, /root/reference/pkg/src) are
called on seeded inputs and their outputs saved, so the GPU box (which has
no /root/reference) can still check parity against the reference.  Complex
right-hand sides use the reference twice (real and imaginary part), valid
because the operator is real.

Each fixture holds: the inputs that are not regenerated cheaply (q), the
tree structure (perm, per-group arrays, list CSR) for bit-exact tree pins,
operator-table checksums, and phi for full / near-only / far-only products.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")


def grid_points(k: int) -> np.ndarray:
    c = (np.arange(k) + 0.5) / k
    xx, yy = np.meshgrid(c, c)
    return np.column_stack((xx.ravel(), yy.ravel()))


def tree_arrays(tree):
    g = tree.groups
    nbr_ptr = np.cumsum([0] + [len(x.neighbors) for x in tree.leaves()])
    nbr_idx = np.array([i for x in tree.leaves() for i in x.neighbors], np.int64)
    int_ptr = np.cumsum([0] + [len(x.interaction) for x in g])
    int_idx = np.array([i for x in g for i in x.interaction], np.int64)
    return dict(
        perm=np.asarray(tree.perm, np.int64),
        level=np.array([x.level for x in g], np.int64),
        ix=np.array([x.ix for x in g], np.int64),
        iy=np.array([x.iy for x in g], np.int64),
        start=np.array([x.start for x in g], np.int64),
        stop=np.array([x.stop for x in g], np.int64),
        parent=np.array([-1 if x.parent is None else x.parent for x in g], np.int64),
        box=np.array([[x.box.xmin, x.box.ymin, x.box.xmax, x.box.ymax] for x in g]),
        nbr_ptr=nbr_ptr.astype(np.int64), nbr_idx=nbr_idx,
        int_ptr=int_ptr.astype(np.int64), int_idx=int_idx,
        meta=np.array([tree.l0, tree.L], np.int64),
        root=np.array([tree.root_origin[0], tree.root_origin[1], tree.root_side]),
    )


def tree_digest(arrs) -> str:
    h = hashlib.sha256()
    for k in sorted(arrs):
        h.update(k.encode())
        h.update(np.ascontiguousarray(arrs[k]).tobytes())
    return h.hexdigest()


def ops_checksums(ops):
    out = {}
    for name in ("V", "U", "C", "B", "D", "near"):
        tab = getattr(ops, name)
        keys = sorted(tab)
        out[f"ops_{name}_sum"] = np.array([float(np.sum(tab[k])) for k in keys])
        out[f"ops_{name}_abs"] = np.array([float(np.sum(np.abs(tab[k]))) for k in keys])
    return out


def make_case(name, pts, P, Q, q, with_dense=True, full_tree=True):
    from taskfmm import dense, fastmvp, operators, quadtree
    tree = quadtree.build_tree(pts, quadtree.TreeParams(P=P))
    ops = operators.build_all(tree, operators.NesaParams(Q=Q))
    q = np.asarray(q)

    def run(**kw):
        if np.iscomplexobj(q):
            return (fastmvp.mvp_serial(tree, ops, q.real.copy(), **kw)
                    + 1j * fastmvp.mvp_serial(tree, ops, q.imag.copy(), **kw))
        return fastmvp.mvp_serial(tree, ops, q, **kw)

    d = dict(points=pts, P=np.int64(P), Q=np.int64(Q), q=q,
             phi=run(), phi_near=run(far=False), phi_far=run(near=False))
    if with_dense:
        if np.iscomplexobj(q):
            d["phi_dense"] = dense.dense_matvec(pts, q.real.copy()) + \
                1j * dense.dense_matvec(pts, q.imag.copy())
        else:
            d["phi_dense"] = dense.dense_matvec(pts, q)
    ta = tree_arrays(tree)
    d["tree_sha256"] = np.array(tree_digest(ta))
    if full_tree:
        d.update({f"tree_{k}": v for k, v in ta.items()})
    d.update(ops_checksums(ops))
    d["task_counts"] = np.array([fastmvp.task_counts(tree)[k] for k in (
        "near", "radiation", "source-transfer", "translation",
        "potential-transfer", "reception")], np.int64)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(f"{name}: N={len(pts)} L={tree.L} G={len(tree.groups)}")


def make_phi_case(name, pts, P, Q, q):
    """A large case stored compactly: the reference's full product only (its
    inputs are regenerated from the seeds), the tree digest and the counts."""
    from taskfmm import fastmvp, operators, quadtree
    tree = quadtree.build_tree(pts, quadtree.TreeParams(P=P))
    ops = operators.build_all(tree, operators.NesaParams(Q=Q))
    phi = (fastmvp.mvp_serial(tree, ops, q.real.copy())
           + 1j * fastmvp.mvp_serial(tree, ops, q.imag.copy()))
    d = dict(P=np.int64(P), Q=np.int64(Q), phi=phi,
             tree_sha256=np.array(tree_digest(tree_arrays(tree))),
             task_counts=np.array([fastmvp.task_counts(tree)[k] for k in (
                 "near", "radiation", "source-transfer", "translation",
                 "potential-transfer", "reception")], np.int64))
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(f"{name}: N={len(pts)} L={tree.L} G={len(tree.groups)}")


def main_c3():
    """BASELINE configs[2] (C3) 2D analog: 200k points on ellipse + plates
    (seed 2), P = 48, Q = 48, complex q (seed 2)."""
    sys.path.insert(0, REF)
    sys.path.insert(0, REPO)
    from paper_1801_03589_b200 import geometry as mine
    n = 200000
    pts = mine.generate_sources(mine.CurveSpec(kind="ellipse-plates", seed=2), n)
    make_phi_case("c3_ellipse_plates_200000", pts, 48, 48, mine.random_rhs(n, 2))


def tree_only(name, pts, P):
    from taskfmm import quadtree
    tree = quadtree.build_tree(pts, quadtree.TreeParams(P=P))
    ta = tree_arrays(tree)
    return name, tree_digest(ta), tree.L, len(tree.groups)


def main():
    sys.path.insert(0, REF)
    sys.path.insert(0, REPO)
    from taskfmm.geometry import CurveSpec, generate_sources
    from paper_1801_03589_b200 import geometry as mine
    os.makedirs(OUT, exist_ok=True)

    wave = lambda n: generate_sources(CurveSpec(), n)  # noqa: E731
    # test_fastmvp.py:54-60 problem
    make_case("fastmvp_1500", wave(1500), 40, 12,
              np.random.default_rng(0).standard_normal(1500))
    # test_fastmvp.py:140-153 single-level tree
    make_case("grid4_single_level", grid_points(4), 16, 14,
              np.random.default_rng(1).standard_normal(16))
    # acceptance criterion 2 (test_acceptance.py:61-76) inputs
    make_case("wave_3000_P50_Q10", wave(3000), 50, 10,
              np.random.default_rng(0).standard_normal(3000), with_dense=False)
    # annulus (acceptance criterion 3 geometry)
    make_case("annulus_1024", generate_sources(
        CurveSpec(kind="annulus-random", seed=1), 1024), 12, 10,
        np.random.default_rng(3).standard_normal(1024))
    # C1: N=2000, leaf 32, Q=24, complex128 q from seed 0
    make_case("c1_wave_2000", wave(2000), 32, 24,
              mine.random_rhs(2000, 0))
    c1 = mine.generate_sources(mine.CurveSpec(kind="circle-random", seed=0), 2000)
    make_case("c1_circle_2000", c1, 32, 24, mine.random_rhs(2000, 0))
    # C2: N=20,000, leaf 32, Q=32, complex q seed 1 (no dense: 20k dense is slow)
    c2 = mine.generate_sources(mine.CurveSpec(kind="circle-random", seed=1), 20000)
    make_case("c2_circle_20000", c2, 32, 32, mine.random_rhs(20000, 1),
              with_dense=False, full_tree=False)
    make_case("c2_wave_20000", wave(20000), 32, 32,
              mine.random_rhs(20000, 1).real.copy(), with_dense=False,
              full_tree=False)
    # C3-like ellipse+plates at reduced N
    ep = mine.generate_sources(mine.CurveSpec(kind="ellipse-plates", seed=2), 20000)
    make_case("ellipse_plates_20000", ep, 48, 48, mine.random_rhs(20000, 2),
              with_dense=False, full_tree=False)

    # Tree digests at the larger configurations (bit-exact tree pins)
    rows = []
    rows.append(tree_only("wave_200000_P48", wave(200000), 48))
    rows.append(tree_only("ellipse_plates_200000_P48", mine.generate_sources(
        mine.CurveSpec(kind="ellipse-plates", seed=2), 200000), 48))
    rows.append(tree_only("circle_random_20000_P32", c2, 32))
    rows.append(tree_only("ellipse_plates_2000000_P64", mine.generate_sources(
        mine.CurveSpec(kind="ellipse-plates", seed=3), 2000000), 64))
    with open(os.path.join(OUT, "tree_digests.txt"), "w") as f:
        for name, dig, L, G in rows:
            f.write(f"{name} {dig} {L} {G}\n")
            print(name, L, G)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "c3":
        main_c3()
    else:
        main()
