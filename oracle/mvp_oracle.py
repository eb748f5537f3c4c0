"""CPU oracle for the NESA matvec -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product path (paper_1801_03589_b200) never
imports it and has no CPU fallback.

It restates the reference's serial product
(/root/reference/pkg/src/taskfmm/fastmvp.py:142-172, ``mvp_serial``) loop for
loop in the same submission order -- near pairs per leaf in neighbor order,
radiation per leaf, source transfer levels L..l0+1, translation levels
l0..L per interaction entry, potential transfer l0+1..L, reception -- with
one generalisation: the work vectors take q's dtype and trailing shape, so
complex128 and multi-RHS (N, m) inputs run through the same loops.  In real
float64 it is bit-identical to the reference (pinned by
tests/test_oracle.py against tests/golden/, which oracle/gen_golden.py made
by running the reference itself).

``dense_matvec`` restates dense.py:14-33 (O(N^2), 512-row chunks).
"""

from __future__ import annotations

import numpy as np

DENSE_CHUNK = 512


def _check_q(tree, q):
    q = np.asarray(q)
    if q.ndim not in (1, 2) or q.shape[0] != tree.n_points:
        raise ValueError("q must have one charge per point")
    return q


def mvp_serial(tree, ops, q, near: bool = True, far: bool = True,
               fraction: float = 1.0):
    """phi = K~ q in the original point order (fastmvp.py:142-172).

    ``fraction`` < 1 runs only the first ceil(fraction * n) iterations of
    every stage loop: the bounded CPU-baseline sample bench.py times.
    """
    q = _check_q(tree, q)
    Q = ops.params.Q
    dt = np.result_type(q.dtype, np.float64)
    tail = q.shape[1:]
    qt = q[tree.perm]
    G = len(tree.groups)
    phi = np.zeros((tree.n_points,) + tail, dt)
    s = np.zeros((G, Q) + tail, dt)
    o = np.zeros((G, Q) + tail, dt)
    groups = tree.groups
    leaves = tree.leaves()

    def cut(seq):
        if fraction >= 1.0:
            return seq
        return seq[:int(np.ceil(fraction * len(seq)))]

    if near:
        for a in cut(leaves):
            for bid in a.neighbors:
                b = groups[bid]
                phi[a.start:a.stop] += ops.near[(a.id, bid)] @ qt[b.start:b.stop]
    if far:
        for b in cut(leaves):
            s[b.id] += ops.V[b.id] @ qt[b.start:b.stop]
        for level in range(tree.L, tree.l0, -1):
            for gid in cut(tree.level_ids[level]):
                s[groups[gid].parent] += ops.C[gid] @ s[gid]
        for level in range(tree.l0, tree.L + 1):
            for aid in cut(tree.level_ids[level]):
                for bid in groups[aid].interaction:
                    o[aid] += ops.D[(aid, bid)] @ s[bid]
        for level in range(tree.l0 + 1, tree.L + 1):
            for gid in cut(tree.level_ids[level]):
                o[gid] += ops.B[gid] @ o[groups[gid].parent]
        for a in cut(leaves):
            phi[a.start:a.stop] += ops.U[a.id] @ o[a.id]
    return phi[tree.inverse_perm()]


def task_counts(tree) -> dict:
    """Per-stage gemv counts (fastmvp.py:175-187)."""
    n_leaves = len(tree.level_ids[tree.L])
    n_edges = sum(len(tree.level_ids[lv]) for lv in range(tree.l0 + 1, tree.L + 1))
    return {
        "near": sum(len(g.neighbors) for g in tree.leaves()),
        "radiation": n_leaves,
        "source-transfer": n_edges,
        "translation": sum(len(g.interaction) for g in tree.groups),
        "potential-transfer": n_edges,
        "reception": n_leaves,
    }


def dense_matvec(points, q):
    """phi_i = sum_{j != i} -log|x_i - x_j| q_j (dense.py:14-33)."""
    points = np.asarray(points, dtype=float)
    q = np.asarray(q)
    n = points.shape[0]
    if q.shape[0] != n:
        raise ValueError("q must have one charge per point")
    phi = np.empty(q.shape, np.result_type(q.dtype, np.float64))
    for a in range(0, n, DENSE_CHUNK):
        b = min(a + DENSE_CHUNK, n)
        diff = points[a:b, None, :] - points[None, :, :]
        d2 = np.einsum("ijk,ijk->ij", diff, diff)
        idx = np.arange(a, b)
        d2[idx - a, idx] = 1.0
        if (d2 == 0.0).any():
            raise ValueError("coincident points")
        phi[a:b] = (-0.5 * np.log(d2)) @ q
    return phi


def near_mask_dense(tree, points_orig):
    """Dense kernel restricted to neighbor-leaf pairs (test_fastmvp.py:42-51)."""
    n = tree.n_points
    mask = np.zeros((n, n), dtype=bool)
    for a in tree.leaves():
        ia = tree.perm[a.start:a.stop]
        for bid in a.neighbors:
            b = tree.groups[bid]
            mask[np.ix_(ia, tree.perm[b.start:b.stop])] = True
    diff = points_orig[:, None, :] - points_orig[None, :, :]
    d2 = np.einsum("ijk,ijk->ij", diff, diff)
    np.fill_diagonal(d2, 1.0)
    return np.where(mask, -0.5 * np.log(d2), 0.0)


def rel_l2(a, b) -> float:
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))
