"""Track B tree checker -- TEST INFRASTRUCTURE ONLY.

A loop-for-loop restatement of the reference's quadtree build
(/root/reference/pkg/src/taskfmm/quadtree.py:123-245) with a third
coordinate: the same stopping rule (140-149), cell arithmetic (111-120),
stable Morton sort (152-157), leaves-first ids and child-run parents
(177-199), 3x3x3 neighbor stencil (214-221) and the parent-neighborhood
interaction rule with Chebyshev distance >= 2 (223-245).  Group objects and
dict lookups exactly as the reference writes them; the product's vectorised
build (paper_1801_03589_b200/octree.py) must reproduce it bit for bit.
The reference itself has no 3D tree, so this restatement is the pin
("parity unpinned" beyond it).
"""

from __future__ import annotations

import numpy as np

MAX_LEVEL = 21


def _morton3(ix, iy, iz):
    key = np.zeros(np.shape(ix), dtype=np.uint64)
    ix = np.asarray(ix).astype(np.uint64)
    iy = np.asarray(iy).astype(np.uint64)
    iz = np.asarray(iz).astype(np.uint64)
    one = np.uint64(1)
    for b in range(MAX_LEVEL):
        bb = np.uint64(b)
        key |= ((ix >> bb) & one) << np.uint64(3 * b)
        key |= ((iy >> bb) & one) << np.uint64(3 * b + 1)
        key |= ((iz >> bb) & one) << np.uint64(3 * b + 2)
    return key


def _cells(points, origin, side, level):
    n_cells = 1 << level
    cell = side / n_cells
    ij = np.floor((points - origin) / cell).astype(np.int64)
    return np.clip(ij, 0, n_cells - 1)


class G3:
    def __init__(self, gid, level, ix, iy, iz, start, stop):
        self.id, self.level, self.ix, self.iy, self.iz = gid, level, ix, iy, iz
        self.start, self.stop = start, stop
        self.parent = None
        self.children = []
        self.neighbors = []
        self.interaction = []


def build_octree_ref(points, P, l0_groups_longest=4):
    """Returns (l0, L, perm, groups, level_ids)."""
    points = np.asarray(points, dtype=float)
    n = points.shape[0]
    lo = points.min(axis=0)
    hi = points.max(axis=0)
    side = float(max(hi - lo))
    origin = lo
    l0 = int(l0_groups_longest).bit_length() - 1

    def count(level):
        c = _cells(points, origin, side, level)
        return np.unique(_morton3(c[:, 0], c[:, 1], c[:, 2])).size

    L = l0
    cnt = count(l0)
    while L < MAX_LEVEL:
        nxt = count(L + 1)
        if nxt <= cnt or n / nxt < P:
            break
        L += 1
        cnt = nxt

    leaf_ij = _cells(points, origin, side, L)
    keys = _morton3(leaf_ij[:, 0], leaf_ij[:, 1], leaf_ij[:, 2])
    perm = np.argsort(keys, kind="stable")
    sk = keys[perm]
    sij = leaf_ij[perm]
    groups, level_ids = [], {}

    def make(level, ix, iy, iz, a, b):
        g = G3(len(groups), level, int(ix), int(iy), int(iz), a, b)
        groups.append(g)
        level_ids.setdefault(level, []).append(g.id)
        return g

    starts = np.flatnonzero(np.r_[True, sk[1:] != sk[:-1]])
    stops = np.r_[starts[1:], n]
    cur = [make(L, *sij[a], int(a), int(b)) for a, b in zip(starts, stops)]
    for level in range(L - 1, l0 - 1, -1):
        nxt = []
        for ch in cur:
            c = (ch.ix >> 1, ch.iy >> 1, ch.iz >> 1)
            if nxt and (nxt[-1].ix, nxt[-1].iy, nxt[-1].iz) == c:
                par = nxt[-1]
                par.stop = ch.stop
            else:
                par = make(level, *c, ch.start, ch.stop)
                nxt.append(par)
            ch.parent = par.id
            par.children.append(ch.id)
        cur = nxt

    cmaps = {lv: {(groups[i].ix, groups[i].iy, groups[i].iz): i for i in ids}
             for lv, ids in level_ids.items()}
    st = [(dx, dy, dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)]
    for gid in level_ids[L]:
        g = groups[gid]
        cm = cmaps[L]
        g.neighbors = sorted(cm[(g.ix + dx, g.iy + dy, g.iz + dz)] for dx, dy, dz in st
                             if (g.ix + dx, g.iy + dy, g.iz + dz) in cm)
    for level in range(l0, L + 1):
        for gid in level_ids[level]:
            g = groups[gid]
            if level == l0:
                cand = level_ids[level]
            else:
                p = groups[g.parent]
                pm = cmaps[level - 1]
                cand = []
                for dx, dy, dz in st:
                    pn = pm.get((p.ix + dx, p.iy + dy, p.iz + dz))
                    if pn is not None:
                        cand.extend(groups[pn].children)
            g.interaction = sorted(
                b for b in cand
                if max(abs(groups[b].ix - g.ix), abs(groups[b].iy - g.iy),
                       abs(groups[b].iz - g.iz)) >= 2)
    return l0, L, perm, groups, level_ids
