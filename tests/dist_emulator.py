"""CPU emulation of one rank's sub-plan -- TEST INFRASTRUCTURE ONLY.

Mirrors what libnesa_b200.so does for NesaPlan(leaf_range=...): stage 1 =
radiation + children-major upward pass over the rank's local groups
(partial sums for groups that straddle ranks), stage 2 = translation,
downward pass, near field and reception for the local leaves.  Loops follow
the reference order (fastmvp.py:142-172) restricted to local work, so with
the exchange of paper_1801_03589_b200.dist the union over ranks equals the
single-device product.
"""

import numpy as np

from paper_1801_03589_b200.dist import local_mask


def stage1(tree, ops, q, leaf_range):
    """Partial s (G, Q) from this rank's leaves."""
    Q = ops.params.Q
    a = tree.arrays
    qt = np.asarray(q)[tree.perm]
    G = a.n_groups
    s = np.zeros((G, Q), dtype=np.result_type(qt.dtype, np.float64))
    mask = local_mask(tree, leaf_range)
    for b in range(*leaf_range):
        s[b] += ops.V[b] @ qt[a.start[b]:a.stop[b]]
    for lv in range(tree.L, tree.l0, -1):
        for c in tree.level_ids[lv]:
            if mask[c]:
                s[a.parent[c]] += ops.C[c] @ s[c]
    return s


def stage2(tree, ops, q, leaf_range, s):
    """phi (N,) with this rank's points filled, zeros elsewhere."""
    Q = ops.params.Q
    a = tree.arrays
    qt = np.asarray(q)[tree.perm]
    G = a.n_groups
    mask = local_mask(tree, leaf_range)
    o = np.zeros((G, Q), dtype=s.dtype)
    for g in np.flatnonzero(mask).tolist():
        for e in range(a.int_ptr[g], a.int_ptr[g + 1]):
            o[g] += ops.D[(g, int(a.int_idx[e]))] @ s[a.int_idx[e]]
    for lv in range(tree.l0 + 1, tree.L + 1):
        for c in tree.level_ids[lv]:
            if mask[c]:
                o[c] += ops.B[c] @ o[a.parent[c]]
    phi_t = np.zeros(tree.n_points, dtype=s.dtype)
    for leaf in range(*leaf_range):
        sl = slice(a.start[leaf], a.stop[leaf])
        for b in a.nbr_idx[a.nbr_ptr[leaf]:a.nbr_ptr[leaf + 1]].tolist():
            phi_t[sl] += ops.near[(leaf, b)] @ qt[a.start[b]:a.stop[b]]
        phi_t[sl] += ops.U[leaf] @ o[leaf]
    phi = np.zeros_like(phi_t)
    lo, hi = a.start[leaf_range[0]], a.stop[leaf_range[1] - 1]
    phi[tree.perm[lo:hi]] = phi_t[lo:hi]
    return phi
