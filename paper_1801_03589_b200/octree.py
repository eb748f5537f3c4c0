"""Sparse uniform-depth octree with neighbor and interaction lists (host).

Track B: the 3D restatement of the reference tree build
(/root/reference/pkg/src/taskfmm/quadtree.py:96-245).  Every rule is the
reference's, carried to three coordinates:

* the root cube's side is the longest bounding-box extent, its corner the
  box minimum (quadtree.py:131-135);
* l0 puts ``l0_groups_longest`` groups along the longest side
  (quadtree.py:137);
* refine while the next level separates some group and the average leaf
  occupancy stays >= P (quadtree.py:140-149);
* cell coordinates ``clip(floor((p - origin) / (side / 2**l)), 0, 2**l - 1)``
  (quadtree.py:111-120); Morton keys interleave x, y, z bits (x lowest);
  the points are stably sorted by the leaf key (quadtree.py:152-157);
* group ids: leaves first in Morton order, then level L-1 ... l0
  (quadtree.py:177-199); a parent's children are consecutive ids;
* leaf neighbors = existing cells of the 3x3x3 stencil, sorted by id;
  interaction lists = at l0 every same-level group, below it the children
  of the parent's 3x3x3 neighborhood, keeping Chebyshev distance >= 2,
  sorted by id (quadtree.py:208-245).

Execution is vectorised numpy over structure-of-arrays (``OctreeArrays``),
the form the GPU plan consumes; ``Group3`` objects are materialised lazily.
``oracle/octree_ref.py`` is the loop-for-loop restatement this build is
pinned against (tests/test_track_b.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .quadtree import TreeParams

MAX_LEVEL = 21          # 3 * 21 = 63 key bits


@dataclass(frozen=True)
class BBox3:
    xmin: float
    ymin: float
    zmin: float
    xmax: float
    ymax: float
    zmax: float

    @property
    def longest_side(self) -> float:
        return max(self.xmax - self.xmin, self.ymax - self.ymin, self.zmax - self.zmin)


def bounding_box3(points: np.ndarray) -> BBox3:
    points = np.asarray(points, dtype=float)
    if points.ndim != 2 or points.shape[1] != 3 or points.shape[0] == 0:
        raise ValueError("points must be a nonempty (n, 3) array")
    lo = points.min(axis=0)
    hi = points.max(axis=0)
    return BBox3(lo[0], lo[1], lo[2], hi[0], hi[1], hi[2])


@dataclass
class Group3:
    """One active box (the 3D Group of quadtree.py:36-68)."""

    id: int
    level: int
    ix: int
    iy: int
    iz: int
    box: BBox3
    parent: int | None = None
    children: list[int] = field(default_factory=list)
    start: int = 0
    stop: int = 0
    neighbors: list[int] = field(default_factory=list)
    interaction: list[int] = field(default_factory=list)

    @property
    def n_points(self) -> int:
        return self.stop - self.start

    @property
    def center(self) -> tuple[float, float, float]:
        b = self.box
        return (0.5 * (b.xmin + b.xmax), 0.5 * (b.ymin + b.ymax), 0.5 * (b.zmin + b.zmax))

    @property
    def half_side(self) -> float:
        return 0.5 * (self.box.xmax - self.box.xmin)

    def is_leaf(self) -> bool:
        return not self.children


@dataclass
class OctreeArrays:
    """Structure-of-arrays octree (group id = array index)."""

    level: np.ndarray        # (G,) int32
    ijk: np.ndarray          # (G, 3) int64 cell coordinates
    start: np.ndarray        # (G,) int64 point range in tree order
    stop: np.ndarray
    parent: np.ndarray       # (G,) int64, -1 at l0
    child_first: np.ndarray  # (G,) int64, -1 for leaves
    n_children: np.ndarray   # (G,) int64
    box: np.ndarray          # (G, 6) xmin, ymin, zmin, xmax, ymax, zmax
    level_first: dict
    level_count: dict
    nbr_ptr: np.ndarray      # (NL+1,) leaf neighbor CSR (sorted ids)
    nbr_idx: np.ndarray
    int_ptr: np.ndarray      # (G+1,) interaction CSR (sorted ids)
    int_idx: np.ndarray

    @property
    def n_groups(self) -> int:
        return int(self.level.shape[0])

    @property
    def ix(self) -> np.ndarray:
        return self.ijk[:, 0]

    @property
    def iy(self) -> np.ndarray:
        return self.ijk[:, 1]

    @property
    def iz(self) -> np.ndarray:
        return self.ijk[:, 2]

    def center(self) -> np.ndarray:
        return 0.5 * (self.box[:, :3] + self.box[:, 3:])

    def half_side(self) -> np.ndarray:
        return 0.5 * (self.box[:, 3] - self.box[:, 0])

    def octant(self) -> np.ndarray:
        """Child kind 4 (ix&1) + 2 (iy&1) + (iz&1): indexes the C / B tables."""
        return (4 * (self.ijk[:, 0] & 1) + 2 * (self.ijk[:, 1] & 1)
                + (self.ijk[:, 2] & 1)).astype(np.int32)


class Octree:
    """Tree object with the reference's attribute names (quadtree.py:71-93)."""

    dim = 3

    def __init__(self, params, l0, L, root_origin, root_side, arrays, perm, points):
        self.params = params
        self.l0 = l0
        self.L = L
        self.root_origin = root_origin
        self.root_side = root_side
        self.arrays: OctreeArrays = arrays
        self.perm = perm
        self.points = points
        self.level_ids = {
            lv: list(range(arrays.level_first[lv], arrays.level_first[lv] + arrays.level_count[lv]))
            for lv in range(L, l0 - 1, -1)
        }
        self._groups = None

    @property
    def n_points(self) -> int:
        return self.points.shape[0]

    @property
    def n_leaves(self) -> int:
        return self.arrays.level_count[self.L]

    @property
    def groups(self) -> list[Group3]:
        if self._groups is None:
            self._groups = _materialize(self.arrays)
        return self._groups

    def leaves(self) -> list[Group3]:
        return [self.groups[i] for i in self.level_ids[self.L]]

    def inverse_perm(self) -> np.ndarray:
        inv = np.empty_like(self.perm)
        inv[self.perm] = np.arange(self.perm.size)
        return inv


def _materialize(a: OctreeArrays) -> list[Group3]:
    out = []
    n_leaves = a.nbr_ptr.shape[0] - 1
    ijk = a.ijk.tolist()
    box = a.box.tolist()
    ip, ii = a.int_ptr.tolist(), a.int_idx.tolist()
    npt, ni = a.nbr_ptr.tolist(), a.nbr_idx.tolist()
    cf, nc = a.child_first.tolist(), a.n_children.tolist()
    for g in range(a.n_groups):
        p = int(a.parent[g])
        out.append(Group3(id=g, level=int(a.level[g]), ix=ijk[g][0], iy=ijk[g][1], iz=ijk[g][2],
                          box=BBox3(*box[g]), parent=None if p < 0 else p,
                          children=list(range(cf[g], cf[g] + nc[g])) if nc[g] else [],
                          start=int(a.start[g]), stop=int(a.stop[g]),
                          neighbors=ni[npt[g]:npt[g + 1]] if g < n_leaves else [],
                          interaction=ii[ip[g]:ip[g + 1]]))
    return out


def morton3(ix, iy, iz) -> np.ndarray:
    """Z-order key: bit b of ix at 3b, of iy at 3b+1, of iz at 3b+2."""

    def dilate(v):
        v = np.asarray(v).astype(np.uint64) & np.uint64(0x1FFFFF)
        for shift, mask in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF),
                            (8, 0x100F00F00F00F00F), (4, 0x10C30C30C30C30C3),
                            (2, 0x1249249249249249)):
            v = (v | (v << np.uint64(shift))) & np.uint64(mask)
        return v

    return dilate(ix) | (dilate(iy) << np.uint64(1)) | (dilate(iz) << np.uint64(2))


def cell_coords3(points, origin, side, level):
    """Integer cell of each point at ``level`` (quadtree.py:111-120 in 3D)."""
    n_cells = 1 << level
    cell = side / n_cells
    ijk = np.floor((points - origin) / cell).astype(np.int64)
    return np.clip(ijk, 0, n_cells - 1)


def _n_cells(points, origin, side, level) -> int:
    c = cell_coords3(points, origin, side, level)
    return int(np.unique(morton3(c[:, 0], c[:, 1], c[:, 2])).size)


_STENCIL3 = np.array([(dx, dy, dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1)
                      for dz in (-1, 0, 1)], dtype=np.int64)


def _lookup(keys_sorted, first_id, c):
    """Group id at integer coords c[..., 3] on one level, -1 where absent."""
    valid = (c >= 0).all(axis=-1)
    cc = np.where(valid[..., None], c, 0)
    k = morton3(cc[..., 0], cc[..., 1], cc[..., 2])
    pos = np.searchsorted(keys_sorted, k)
    pos_c = np.minimum(pos, keys_sorted.size - 1)
    hit = valid & (pos < keys_sorted.size) & (keys_sorted[pos_c] == k)
    return np.where(hit, first_id + pos_c, -1)


def _rows_to_csr(cand):
    big = np.iinfo(np.int64).max
    c = np.where(cand < 0, big, cand)
    c.sort(axis=1)
    cnt = (c != big).sum(axis=1)
    ptr = np.zeros(cand.shape[0] + 1, np.int64)
    np.cumsum(cnt, out=ptr[1:])
    return ptr, c[c != big].astype(np.int64)


def build_octree(points: np.ndarray, params: TreeParams) -> Octree:
    """Build the octree and its lists (quadtree.py:123-245 in 3D)."""
    points = np.ascontiguousarray(points, dtype=float)
    if points.ndim != 2 or points.shape[1] != 3 or points.shape[0] == 0:
        raise ValueError("points must be a nonempty (n, 3) array")
    n = points.shape[0]
    if n < params.l0_groups_longest:
        raise ValueError("too few points for the coarsest level")
    if np.unique(points, axis=0).shape[0] != n:
        raise ValueError("points must be pairwise distinct")
    bb = bounding_box3(points)
    side = bb.longest_side
    if side <= 0:
        raise ValueError("degenerate point set (zero extent)")
    origin = np.array([bb.xmin, bb.ymin, bb.zmin])
    l0 = int(params.l0_groups_longest).bit_length() - 1

    L = l0
    count = _n_cells(points, origin, side, l0)
    while L < MAX_LEVEL:
        nxt = _n_cells(points, origin, side, L + 1)
        if nxt <= count or n / nxt < params.P:
            break
        L += 1
        count = nxt

    leaf = cell_coords3(points, origin, side, L)
    keys = morton3(leaf[:, 0], leaf[:, 1], leaf[:, 2])
    perm = np.argsort(keys, kind="stable")
    skeys = keys[perm]
    brk = np.flatnonzero(np.r_[True, skeys[1:] != skeys[:-1]])
    lvl_keys = {L: skeys[brk]}
    lvl_start = {L: brk.astype(np.int64)}
    lvl_ijk = {L: leaf[perm[brk]]}
    lvl_parent_local = {}
    for lv in range(L - 1, l0 - 1, -1):
        ck = lvl_keys[lv + 1] >> np.uint64(3)
        first = np.r_[True, ck[1:] != ck[:-1]]
        pos = np.flatnonzero(first)
        lvl_parent_local[lv + 1] = np.cumsum(first) - 1
        lvl_keys[lv] = ck[pos]
        lvl_start[lv] = lvl_start[lv + 1][pos]
        lvl_ijk[lv] = lvl_ijk[lv + 1][pos] >> 1

    level_first, level_count = {}, {}
    nid = 0
    for lv in range(L, l0 - 1, -1):
        level_first[lv] = nid
        level_count[lv] = int(lvl_keys[lv].size)
        nid += level_count[lv]
    G = nid
    level = np.empty(G, np.int32)
    ijk = np.empty((G, 3), np.int64)
    start = np.empty(G, np.int64)
    stop = np.empty(G, np.int64)
    parent = np.full(G, -1, np.int64)
    child_first = np.full(G, -1, np.int64)
    n_children = np.zeros(G, np.int64)
    box = np.empty((G, 6))
    for lv in range(L, l0 - 1, -1):
        s = slice(level_first[lv], level_first[lv] + level_count[lv])
        level[s] = lv
        ijk[s] = lvl_ijk[lv]
        start[s] = lvl_start[lv]
        stop[s] = np.r_[lvl_start[lv][1:], n]
        h = side / (1 << lv)
        box[s, :3] = origin + ijk[s] * h
        box[s, 3:] = origin + (ijk[s] + 1) * h
        if lv > l0:
            pid = level_first[lv - 1] + lvl_parent_local[lv]
            parent[s] = pid
            ids = np.arange(level_first[lv], level_first[lv] + level_count[lv])
            f = np.r_[True, pid[1:] != pid[:-1]]
            child_first[pid[f]] = ids[f]
            n_children += np.bincount(pid, minlength=G)

    a = OctreeArrays(level=level, ijk=ijk, start=start, stop=stop, parent=parent,
                     child_first=child_first, n_children=n_children, box=box,
                     level_first=level_first, level_count=level_count,
                     nbr_ptr=None, nbr_idx=None, int_ptr=None, int_idx=None)
    _fill_lists(a, lvl_keys, L, l0)
    return Octree(params=params, l0=l0, L=L, root_origin=tuple(float(v) for v in origin),
                  root_side=side, arrays=a, perm=perm, points=points[perm])


def _fill_lists(a: OctreeArrays, lvl_keys, L, l0) -> None:
    G = a.n_groups
    s = slice(a.level_first[L], a.level_first[L] + a.level_count[L])
    cand = _lookup(lvl_keys[L], a.level_first[L], a.ijk[s][:, None, :] + _STENCIL3[None])
    a.nbr_ptr, a.nbr_idx = _rows_to_csr(cand)
    counts = np.zeros(G, np.int64)
    rows = {}
    for lv in range(l0, L + 1):
        f, c = a.level_first[lv], a.level_count[lv]
        ids = np.arange(f, f + c)
        if lv == l0:
            cand = np.broadcast_to(ids, (c, c)).copy()
        else:
            p = a.parent[ids]
            pn = _lookup(lvl_keys[lv - 1], a.level_first[lv - 1],
                         a.ijk[p][:, None, :] + _STENCIL3[None])          # (c, 27)
            cf = np.where(pn >= 0, a.child_first[np.maximum(pn, 0)], -1)
            nc = np.where(pn >= 0, a.n_children[np.maximum(pn, 0)], 0)
            k = np.arange(8)
            cand = np.where(k[None, None, :] < nc[:, :, None],
                            cf[:, :, None] + k[None, None, :], -1).reshape(c, 27 * 8)
        safe = np.maximum(cand, 0)
        cheb = np.abs(a.ijk[safe] - a.ijk[ids][:, None, :]).max(axis=-1)
        cand = np.where((cand >= 0) & (cheb >= 2), cand, -1)
        ptr, idx = _rows_to_csr(cand)
        rows[lv] = idx
        counts[ids] = np.diff(ptr)
    a.int_ptr = np.zeros(G + 1, np.int64)
    np.cumsum(counts, out=a.int_ptr[1:])
    a.int_idx = np.concatenate([rows[lv] for lv in range(L, l0 - 1, -1)])


def octree_stats(tree: Octree) -> dict:
    a = tree.arrays
    counts = {lv: a.level_count[lv] for lv in range(tree.l0, tree.L + 1)}
    isz = np.diff(a.int_ptr)
    return {
        "levels": list(range(tree.l0, tree.L + 1)),
        "groups_per_level": counts,
        "n_leaves": counts[tree.L],
        "avg_neighbors": float(np.mean(np.diff(a.nbr_ptr))),
        "avg_interaction": float(np.mean(isz)),
        "max_interaction": int(isz.max()) if isz.size else 0,
        "avg_leaf_points": tree.n_points / counts[tree.L],
    }
