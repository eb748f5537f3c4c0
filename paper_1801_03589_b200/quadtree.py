"""Sparse uniform-depth quadtree with neighbor and interaction lists (host).

Bit-exact restatement of the reference tree build
(/root/reference/pkg/src/taskfmm/quadtree.py:96-245): the same stopping
rule, cell-coordinate arithmetic (true division by ``side / 2**level``,
floor, clip), stable Morton sort, leaves-first group ids and id-sorted
lists.  What differs is the execution: every step is a vectorised numpy
pass over structure-of-arrays (``TreeArrays``), which is also the form the
GPU plan consumes, and the reference-style ``Group`` objects are
materialised lazily for callers that walk ``tree.groups``.

Public surface mirrors the reference: ``TreeParams``, ``Group``, ``Tree``,
``build_tree``, ``neighbor_list``, ``interaction_list``, ``tree_stats``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .geometry import BBox, bounding_box

MAX_LEVEL = 30


@dataclass(frozen=True)
class TreeParams:
    """P is the target average number of points per leaf (quadtree.py:21-33)."""

    P: int = 50
    l0_groups_longest: int = 4

    def __post_init__(self):
        if self.P < 1:
            raise ValueError("P must be >= 1")
        k = self.l0_groups_longest
        if k < 2 or (k & (k - 1)) != 0:
            raise ValueError("l0_groups_longest must be a power of two >= 2")


@dataclass
class Group:
    """One active box (quadtree.py:36-68)."""

    id: int
    level: int
    ix: int
    iy: int
    box: BBox
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
    def center(self) -> tuple[float, float]:
        return (0.5 * (self.box.xmin + self.box.xmax),
                0.5 * (self.box.ymin + self.box.ymax))

    @property
    def half_side(self) -> float:
        return 0.5 * (self.box.xmax - self.box.xmin)

    def is_leaf(self) -> bool:
        return not self.children


@dataclass
class TreeArrays:
    """Structure-of-arrays form of the tree (group id = array index).

    Ids are leaves first (level L, Morton order), then level L-1, ... l0,
    each level a contiguous id range ``level_start[l - l0] ..`` in Morton
    order, exactly as quadtree.py:177-199 assigns them.
    """

    level: np.ndarray        # (G,) int32
    ix: np.ndarray           # (G,) int64
    iy: np.ndarray           # (G,) int64
    start: np.ndarray        # (G,) int64 point range in tree order
    stop: np.ndarray         # (G,) int64
    parent: np.ndarray       # (G,) int64, -1 at l0
    child_first: np.ndarray  # (G,) int64, first child id (-1 for leaves)
    n_children: np.ndarray   # (G,) int64
    box: np.ndarray          # (G, 4) float64 xmin, ymin, xmax, ymax
    level_first: dict        # level -> first id of that level
    level_count: dict        # level -> number of groups
    nbr_ptr: np.ndarray      # (NL+1,) CSR of leaf neighbor lists (sorted ids)
    nbr_idx: np.ndarray
    int_ptr: np.ndarray      # (G+1,) CSR of interaction lists (sorted ids)
    int_idx: np.ndarray

    @property
    def n_groups(self) -> int:
        return int(self.level.shape[0])

    def center(self) -> np.ndarray:
        return np.column_stack((0.5 * (self.box[:, 0] + self.box[:, 2]),
                                0.5 * (self.box[:, 1] + self.box[:, 3])))

    def half_side(self) -> np.ndarray:
        return 0.5 * (self.box[:, 2] - self.box[:, 0])


class Tree:
    """Reference-compatible tree object (quadtree.py:71-93) over TreeArrays."""

    def __init__(self, params, l0, L, root_origin, root_side, arrays, perm, points):
        self.params = params
        self.l0 = l0
        self.L = L
        self.root_origin = root_origin
        self.root_side = root_side
        self.arrays: TreeArrays = arrays
        self.perm = perm
        self.points = points
        self.level_ids = {
            lv: list(range(arrays.level_first[lv],
                           arrays.level_first[lv] + arrays.level_count[lv]))
            for lv in range(L, l0 - 1, -1)
        }
        self._groups = None
        self._inv = None

    @property
    def n_points(self) -> int:
        return self.points.shape[0]

    @property
    def n_leaves(self) -> int:
        return self.arrays.level_count[self.L]

    @property
    def groups(self) -> list[Group]:
        if self._groups is None:
            self._groups = _materialize_groups(self.arrays)
        return self._groups

    def leaves(self) -> list[Group]:
        return [self.groups[i] for i in self.level_ids[self.L]]

    def inverse_perm(self) -> np.ndarray:
        if self._inv is None:
            inv = np.empty_like(self.perm)
            inv[self.perm] = np.arange(self.perm.size)
            self._inv = inv
        return self._inv.copy()


def _materialize_groups(a: TreeArrays) -> list[Group]:
    G = a.n_groups
    lvl = a.level.tolist()
    ix = a.ix.tolist()
    iy = a.iy.tolist()
    st = a.start.tolist()
    sp = a.stop.tolist()
    par = a.parent.tolist()
    cf = a.child_first.tolist()
    nc = a.n_children.tolist()
    box = a.box.tolist()
    ip = a.int_ptr.tolist()
    ii = a.int_idx.tolist()
    npt = a.nbr_ptr.tolist()
    ni = a.nbr_idx.tolist()
    n_leaves = len(npt) - 1
    out = []
    for g in range(G):
        grp = Group(id=g, level=lvl[g], ix=ix[g], iy=iy[g], box=BBox(*box[g]),
                    parent=None if par[g] < 0 else par[g],
                    children=list(range(cf[g], cf[g] + nc[g])) if nc[g] else [],
                    start=st[g], stop=sp[g],
                    neighbors=ni[npt[g]:npt[g + 1]] if g < n_leaves else [],
                    interaction=ii[ip[g]:ip[g + 1]])
        out.append(grp)
    return out


def _morton(ix: np.ndarray, iy: np.ndarray) -> np.ndarray:
    """Z-order key: bits of ix at even positions, iy at odd (quadtree.py:96-108)."""

    def dilate(v):
        v = np.asarray(v).astype(np.uint64)
        for shift, mask in ((16, 0x0000FFFF0000FFFF), (8, 0x00FF00FF00FF00FF),
                            (4, 0x0F0F0F0F0F0F0F0F), (2, 0x3333333333333333),
                            (1, 0x5555555555555555)):
            v = (v | (v << np.uint64(shift))) & np.uint64(mask)
        return v

    return dilate(ix) | (dilate(iy) << np.uint64(1))


def _cell_coords(points, origin, side, level):
    """Integer cell of each point at ``level`` (quadtree.py:111-120)."""
    n_cells = 1 << level
    cell = side / n_cells
    ij = np.floor((points - origin) / cell).astype(np.int64)
    return np.clip(ij, 0, n_cells - 1)


def _n_cells_used(points, origin, side, level) -> int:
    ij = _cell_coords(points, origin, side, level)
    return int(np.unique(_morton(ij[:, 0], ij[:, 1])).size)


def _lookup(keys_sorted: np.ndarray, first_id: int, qx, qy) -> np.ndarray:
    """Group id at integer coords (qx, qy) on one level, -1 where absent."""
    valid = (qx >= 0) & (qy >= 0)
    k = _morton(np.where(valid, qx, 0), np.where(valid, qy, 0))
    pos = np.searchsorted(keys_sorted, k)
    pos_c = np.minimum(pos, keys_sorted.size - 1)
    hit = valid & (pos < keys_sorted.size) & (keys_sorted[pos_c] == k)
    return np.where(hit, first_id + pos_c, -1)


def _sorted_rows_to_csr(cand: np.ndarray):
    """Rows of candidate ids (-1 = none) -> CSR with each row sorted ascending."""
    big = np.iinfo(np.int64).max
    c = np.where(cand < 0, big, cand)
    c.sort(axis=1)
    cnt = (c != big).sum(axis=1)
    ptr = np.zeros(cand.shape[0] + 1, dtype=np.int64)
    np.cumsum(cnt, out=ptr[1:])
    idx = c[c != big].astype(np.int64)   # row-major order keeps rows contiguous
    return ptr, idx


def _build_tree_native(points: np.ndarray, params: TreeParams):
    """The same build in C++ (csrc/nesa_tree.cpp via the C ABI); None when
    the library is not built.  Bit-identical arrays (tests/test_host_tree.py)."""
    import ctypes
    try:
        from . import _capi
        lib = _capi.load()
    except (OSError, RuntimeError):
        return None
    n = points.shape[0]
    h = ctypes.c_void_p()
    rc = lib.nesa_tree_build(points.ctypes.data, n, float(params.P), int(params.l0_groups_longest),
                             ctypes.byref(h))
    try:
        if rc != 0:
            msg = lib.nesa_tree_error(h).decode()
            if rc == 1:
                raise ValueError(msg)
            raise RuntimeError(msg)
        size = lambda w: int(lib.nesa_tree_size(h, w))  # noqa: E731
        G, NL, nn, ni, l0, L = (size(w) for w in range(6))

        def get(field, count, dtype, shape=None):
            out = np.empty(count, dtype)
            if count:
                lib.nesa_tree_copy(h, field, out.ctypes.data)
            return out if shape is None else out.reshape(shape)

        nlev = L - l0 + 1
        lf = get(9, nlev, np.int64)
        lc = get(10, nlev, np.int64)
        geo = get(16, 3, np.float64)
        arrays = TreeArrays(level=get(0, G, np.int32), ix=get(1, G, np.int64), iy=get(2, G, np.int64),
                            start=get(3, G, np.int64), stop=get(4, G, np.int64),
                            parent=get(5, G, np.int64), child_first=get(6, G, np.int64),
                            n_children=get(7, G, np.int64), box=get(8, 4 * G, np.float64, (G, 4)),
                            level_first={l0 + i: int(lf[i]) for i in range(nlev)},
                            level_count={l0 + i: int(lc[i]) for i in range(nlev)},
                            nbr_ptr=get(11, NL + 1, np.int64), nbr_idx=get(12, nn, np.int64),
                            int_ptr=get(13, G + 1, np.int64), int_idx=get(14, ni, np.int64))
        perm = get(15, n, np.int64)
    finally:
        lib.nesa_tree_free(h)
    return Tree(params=params, l0=l0, L=L, root_origin=(float(geo[0]), float(geo[1])),
                root_side=float(geo[2]), arrays=arrays, perm=perm, points=points[perm])


def build_tree(points: np.ndarray, params: TreeParams, native: bool | None = None) -> Tree:
    """Build the quadtree and its lists (quadtree.py:123-205).

    ``native`` (default: the C++ build when the library is built,
    NESA_TREE_NATIVE=0 forces numpy) selects csrc/nesa_tree.cpp; both give
    bit-identical trees.
    """
    import os
    points = np.ascontiguousarray(points, dtype=float)
    if points.ndim != 2 or points.shape[1] != 2 or points.shape[0] == 0:
        raise ValueError("points must be a nonempty (n, 2) array")
    if native is None:
        native = os.environ.get("NESA_TREE_NATIVE", "1") != "0"
    if native:
        t = _build_tree_native(points, params)
        if t is not None:
            return t
    return _build_tree_numpy(points, params)


def _build_tree_numpy(points: np.ndarray, params: TreeParams) -> Tree:
    n = points.shape[0]
    if n < params.l0_groups_longest:
        raise ValueError("too few points for the coarsest level")
    # distinct rows <=> distinct complex numbers x + iy (one 1-D sort instead
    # of np.unique(axis=0)'s row sort: 0.25 s instead of 1.75 s at 2M points)
    if np.unique(points.view(np.complex128).ravel()).size != n:
        raise ValueError("points must be pairwise distinct")
    bb = bounding_box(points)
    side = bb.longest_side
    if side <= 0:
        raise ValueError("degenerate point set (zero extent)")
    origin = np.array([bb.xmin, bb.ymin])
    l0 = int(params.l0_groups_longest).bit_length() - 1

    # Stopping rule: refine while the next level splits some group and the
    # average occupancy stays >= P (quadtree.py:140-149).
    L = l0
    count = _n_cells_used(points, origin, side, l0)
    while L < MAX_LEVEL:
        nxt = _n_cells_used(points, origin, side, L + 1)
        if nxt <= count or n / nxt < params.P:
            break
        L += 1
        count = nxt

    leaf_ij = _cell_coords(points, origin, side, L)
    keys = _morton(leaf_ij[:, 0], leaf_ij[:, 1])
    perm = np.argsort(keys, kind="stable")
    skeys = keys[perm]
    tpoints = points[perm]

    # Per level (fine -> coarse): Morton-sorted unique cells with point ranges.
    brk = np.flatnonzero(np.r_[True, skeys[1:] != skeys[:-1]])
    lvl_keys = {L: skeys[brk]}
    lvl_start = {L: brk.astype(np.int64)}
    lvl_stop = {L: np.r_[brk[1:], n].astype(np.int64)}
    lvl_ij = {L: leaf_ij[perm[brk]]}
    lvl_parent_local = {}
    for lv in range(L - 1, l0 - 1, -1):
        ck = lvl_keys[lv + 1] >> np.uint64(2)     # parent key of each child
        first = np.r_[True, ck[1:] != ck[:-1]]
        pos = np.flatnonzero(first)
        lvl_parent_local[lv + 1] = np.cumsum(first) - 1
        lvl_keys[lv] = ck[pos]
        lvl_start[lv] = lvl_start[lv + 1][pos]
        lvl_stop[lv] = np.r_[lvl_start[lv + 1][pos[1:]], n].astype(np.int64)
        lvl_ij[lv] = lvl_ij[lv + 1][pos] >> 1

    level_first, level_count = {}, {}
    nxt_id = 0
    for lv in range(L, l0 - 1, -1):
        level_first[lv] = nxt_id
        level_count[lv] = int(lvl_keys[lv].size)
        nxt_id += level_count[lv]
    G = nxt_id

    level = np.empty(G, np.int32)
    ix = np.empty(G, np.int64)
    iy = np.empty(G, np.int64)
    start = np.empty(G, np.int64)
    stop = np.empty(G, np.int64)
    parent = np.full(G, -1, np.int64)
    child_first = np.full(G, -1, np.int64)
    n_children = np.zeros(G, np.int64)
    box = np.empty((G, 4))
    for lv in range(L, l0 - 1, -1):
        s = slice(level_first[lv], level_first[lv] + level_count[lv])
        level[s] = lv
        ix[s] = lvl_ij[lv][:, 0]
        iy[s] = lvl_ij[lv][:, 1]
        start[s] = lvl_start[lv]
        stop[s] = lvl_stop[lv]
        h = side / (1 << lv)
        box[s, 0] = origin[0] + ix[s] * h
        box[s, 1] = origin[1] + iy[s] * h
        box[s, 2] = origin[0] + (ix[s] + 1) * h
        box[s, 3] = origin[1] + (iy[s] + 1) * h
        if lv > l0:
            pid = level_first[lv - 1] + lvl_parent_local[lv]
            parent[s] = pid
            ids = np.arange(level_first[lv], level_first[lv] + level_count[lv])
            first = np.r_[True, pid[1:] != pid[:-1]]
            child_first[pid[first]] = ids[first]
            n_children[:] += np.bincount(pid, minlength=G)

    arrays = TreeArrays(level=level, ix=ix, iy=iy, start=start, stop=stop,
                        parent=parent, child_first=child_first,
                        n_children=n_children, box=box,
                        level_first=level_first, level_count=level_count,
                        nbr_ptr=None, nbr_idx=None, int_ptr=None, int_idx=None)
    _fill_lists(arrays, lvl_keys, L, l0)
    return Tree(params=params, l0=l0, L=L, root_origin=(origin[0], origin[1]),
                root_side=side, arrays=arrays, perm=perm, points=tpoints)


_STENCIL = np.array([(dx, dy) for dx in (-1, 0, 1) for dy in (-1, 0, 1)])


def _fill_lists(a: TreeArrays, lvl_keys, L, l0) -> None:
    """Neighbor lists (leaves) and interaction lists (quadtree.py:208-245)."""
    G = a.n_groups
    # Leaf neighbors: existing cells of the 3x3 stencil, sorted by id.
    s = slice(a.level_first[L], a.level_first[L] + a.level_count[L])
    gx, gy = a.ix[s], a.iy[s]
    cand = _lookup(lvl_keys[L], a.level_first[L],
                   gx[:, None] + _STENCIL[None, :, 0],
                   gy[:, None] + _STENCIL[None, :, 1])
    a.nbr_ptr, a.nbr_idx = _sorted_rows_to_csr(cand)

    counts = np.zeros(G, np.int64)
    rows = {}
    for lv in range(l0, L + 1):
        f, c = a.level_first[lv], a.level_count[lv]
        ids = np.arange(f, f + c)
        if lv == l0:
            cand = np.broadcast_to(ids, (c, c)).copy()
        else:
            # children of the 3x3 parent-level neighborhood of the parent
            p = a.parent[ids]
            pn = _lookup(lvl_keys[lv - 1], a.level_first[lv - 1],
                         a.ix[p][:, None] + _STENCIL[None, :, 0],
                         a.iy[p][:, None] + _STENCIL[None, :, 1])   # (c, 9)
            cf = np.where(pn >= 0, a.child_first[np.maximum(pn, 0)], -1)
            nc = np.where(pn >= 0, a.n_children[np.maximum(pn, 0)], 0)
            k = np.arange(4)
            cand = np.where(k[None, None, :] < nc[:, :, None],
                            cf[:, :, None] + k[None, None, :], -1).reshape(c, 36)
        safe = np.maximum(cand, 0)
        cheb = np.maximum(np.abs(a.ix[safe] - a.ix[ids][:, None]),
                          np.abs(a.iy[safe] - a.iy[ids][:, None]))
        cand = np.where((cand >= 0) & (cheb >= 2), cand, -1)
        ptr, idx = _sorted_rows_to_csr(cand)
        rows[lv] = (ptr, idx)
        counts[ids] = np.diff(ptr)
    # Concatenate per-level CSR in id order (levels are contiguous id ranges,
    # finest level first).
    a.int_ptr = np.zeros(G + 1, np.int64)
    np.cumsum(counts, out=a.int_ptr[1:])
    a.int_idx = np.concatenate([rows[lv][1] for lv in range(L, l0 - 1, -1)]) \
        if G else np.zeros(0, np.int64)


def neighbor_list(tree: Tree, g: Group) -> list[Group]:
    """Same-level groups touching a leaf, itself included (quadtree.py:248-252)."""
    if not g.is_leaf():
        raise ValueError("neighbor lists are defined for leaves only")
    return [tree.groups[i] for i in g.neighbors]


def interaction_list(tree: Tree, g: Group) -> list[Group]:
    """Far-field partners of g at its own level (quadtree.py:255-257)."""
    return [tree.groups[i] for i in g.interaction]


def tree_stats(tree: Tree) -> dict:
    """Occupancy and list-size statistics (quadtree.py:260-281)."""
    a = tree.arrays
    counts = {lv: a.level_count[lv] for lv in range(tree.l0, tree.L + 1)}
    n_parents = sum(counts[lv] for lv in range(tree.l0, tree.L))
    n_children = sum(counts[lv] for lv in range(tree.l0 + 1, tree.L + 1))
    isz = np.diff(a.int_ptr)
    per_level = {}
    for lv in range(tree.l0, tree.L + 1):
        f, c = a.level_first[lv], a.level_count[lv]
        per_level[lv] = float(np.mean(isz[f:f + c]))
    return {
        "levels": list(range(tree.l0, tree.L + 1)),
        "groups_per_level": counts,
        "n_leaves": counts[tree.L],
        "n_transfer_edges": n_children,
        "avg_children": (n_children / n_parents) if n_parents else 0.0,
        "avg_neighbors": float(np.mean(np.diff(a.nbr_ptr))),
        "avg_interaction": float(np.mean(isz)),
        "avg_interaction_per_level": per_level,
        "avg_leaf_points": tree.n_points / counts[tree.L],
    }
