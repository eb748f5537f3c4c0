"""Track B golden fixtures from the REFERENCE's own product -- TEST INFRASTRUCTURE.

The reference cannot build 3D / Helmholtz operators, but its serial product
(/root/reference/pkg/src/taskfmm/fastmvp.py:142-172, ``mvp_serial``) is
generic over the tree and operator containers: it walks ``tree.leaves()``,
``groups[...].neighbors / .interaction / .parent / .start / .stop`` and
``level_ids``, and multiplies the dict matrices into float64 stage vectors.
A complex Track B problem in its real 2x2 embedding (every complex entry
a + ib -> [[a, -b], [b, a]], point ranges and Q doubled, q viewed as 2N
reals) is therefore a problem the reference's code computes as it is.  This
script builds Track B problems with our octree / Helmholtz operators
(paper_1801_03589_b200.octree / .helmholtz), runs the reference's
``mvp_serial`` on the embedded form, and stores q and phi (complex) as
``tests/golden/track_b_*.npz`` -- the pin for the dtype-generic oracle and,
through it, for the GPU product (tests/test_track_b.py).

    python oracle/gen_golden_track_b.py      (needs /root/reference; run here, not on the GPU box)
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
REF = "/root/reference/pkg/src"

CASES = {
    # name: (surface, n, seed, leaf P, Q, wavenumber or None for 10 points per wavelength)
    "track_b_sphere_2000": ("sphere", 2000, 0, 32, 24, None),
    "track_b_sphere_6000_levels": ("sphere", 6000, 7, 8, 16, 3.0),
    "track_b_ellipsoid_plates_8000": ("ellipsoid-plates", 8000, 2, 16, 16, None),
}


class _EGroup:
    def __init__(self, g):
        self.id = g.id
        self.level = g.level
        self.start = 2 * g.start
        self.stop = 2 * g.stop
        self.parent = g.parent
        self.children = g.children
        self.neighbors = g.neighbors
        self.interaction = g.interaction


class _ETree:
    """The octree seen by the reference's mvp_serial in the real embedding."""

    def __init__(self, tree):
        self.groups = [_EGroup(g) for g in tree.groups]
        self.level_ids = tree.level_ids
        self.L, self.l0 = tree.L, tree.l0
        self.perm = (2 * tree.perm[:, None] + np.arange(2)[None, :]).reshape(-1)
        self.n_points = 2 * tree.n_points

    def leaves(self):
        return [self.groups[i] for i in self.level_ids[self.L]]

    def inverse_perm(self):
        inv = np.empty_like(self.perm)
        inv[self.perm] = np.arange(self.perm.size)
        return inv


class _EParams:
    def __init__(self, Q):
        self.Q = Q


class _EOps:
    def __init__(self, ops):
        from paper_1801_03589_b200.plan3 import embed
        self.params = _EParams(2 * ops.params.Q)
        cache = {}

        def e(m):   # shared objects stay shared (the reference's dict semantics)
            key = id(m)
            if key not in cache:
                cache[key] = embed(m)
            return cache[key]
        self.near = {k: e(v) for k, v in ops.near.items()}
        self.V = {k: e(v) for k, v in ops.V.items()}
        self.U = {k: e(v) for k, v in ops.U.items()}
        self.C = {k: e(v) for k, v in ops.C.items()}
        self.B = {k: e(v) for k, v in ops.B.items()}
        self.D = {k: e(v) for k, v in ops.D.items()}


def reference_product(tree, ops, q, near=True, far=True):
    """phi = K~ q (complex) computed by the reference's mvp_serial on the embedding."""
    sys.path.insert(0, REF)
    from taskfmm.fastmvp import mvp_serial as ref_mvp
    qe = np.ascontiguousarray(q, dtype=np.complex128).view(np.float64)
    phi = ref_mvp(_ETree(tree), _EOps(ops), qe, near=near, far=far)
    return np.ascontiguousarray(phi).view(np.complex128)


def build_case(name):
    from paper_1801_03589_b200 import helmholtz as hz
    from paper_1801_03589_b200.octree import build_octree
    from paper_1801_03589_b200.quadtree import TreeParams
    kind, n, seed, P, Q, k = CASES[name]
    pts = hz.generate_surface(kind, n, seed)
    tree = build_octree(pts, TreeParams(P=P))
    params = hz.HelmholtzParams(Q=Q, k=k if k is not None else hz.wavenumber3(kind, n))
    rng = np.random.default_rng(seed)
    q = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return pts, tree, params, q


def main():
    from paper_1801_03589_b200 import helmholtz as hz
    out_dir = os.path.join(HERE, "tests", "golden")
    for name in CASES:
        pts, tree, params, q = build_case(name)
        ops = hz.build_all3(tree, params)
        phi = reference_product(tree, ops, q)
        phi_near = reference_product(tree, ops, q, far=False)
        np.savez_compressed(os.path.join(out_dir, f"{name}.npz"), q=q, phi=phi, phi_near=phi_near,
                            k=params.k, Q=params.Q, levels=tree.L - tree.l0 + 1)
        print(name, tree.L - tree.l0 + 1, "levels", f"|phi| {np.linalg.norm(phi):.4e}", flush=True)


if __name__ == "__main__":
    main()
