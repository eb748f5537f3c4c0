"""Track B host side: 3D surfaces, the Helmholtz kernel and complex operators.

BASELINE.json's configurations are literally 3D (sphere; ellipsoid + plates)
with a Helmholtz kernel and complex operators; the reference is 2D, real and
log-kernel only.  This module restates the reference's
operator construction (/root/reference/pkg/src/taskfmm/operators.py:34-253)
with three substitutions and nothing else:

* the kernel is G(x, y) = exp(-j k |x - y|) / (4 pi |x - y|) (zero on the
  diagonal of a same-set block, an error for coincident distinct points --
  linalg.py:22-44's rules);
* the auxiliary / check circles become spheres of ``count`` points on a
  Fibonacci lattice (deterministic, near-uniform), radii rho * h as before;
* the tree is the octree (octree.py): C / B are cached per (level, child
  octant), D per (level, integer 3D offset) -- translation invariance holds
  for the Helmholtz kernel exactly as for the log kernel.

The equivalent-source fits are the reference's truncated-SVD pseudoinverse
(linalg.py:56-67) of the complex aux -> check matrices.  The geometry ratios
are the reference's constraints carried to 3D (sqrt(3) for the box's
half-diagonal instead of sqrt(2)).

The product on these operators is pinned against the reference's own
mvp_serial run on their real embedding (oracle/gen_golden_track_b.py,
tests/golden/track_b_*.npz); the operator construction itself is ours --
the reference cannot produce 3D / Helmholtz operators.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .octree import Octree
from .quadtree import TreeParams

SQRT3 = math.sqrt(3.0)
ELLIPSOID_AXES = (5.0, 0.5, 0.5)
PLATE_SIZE = (4.0, 1.0)        # x extent, y extent
PLATE_Z = 1.5                  # plates in the planes z = +-1.5 (builder's choice)


# ----------------------------------------------------------------------------
# geometry
# ----------------------------------------------------------------------------
def sphere_surface(n: int, seed: int) -> np.ndarray:
    """n points uniform on the unit sphere: normalised N(0, I) draws."""
    v = np.random.default_rng(seed).standard_normal((n, 3))
    return v / np.linalg.norm(v, axis=1)[:, None]


def spheroid_area(a: float, b: float) -> float:
    """Surface area of the prolate spheroid with semi-axes (a, b, b), a > b."""
    e = math.sqrt(1.0 - (b / a) ** 2)
    return 2.0 * math.pi * b * b * (1.0 + a / (b * e) * math.asin(e))


def _ellipsoid_surface(n: int, rng) -> np.ndarray:
    """Area-uniform points on the ellipsoid (a, b, c): uniform sphere draws
    mapped by diag(a, b, c), accepted with probability proportional to the
    map's area element |(bc u_x, ac u_y, ab u_z)| (rejection, in order)."""
    a, b, c = ELLIPSOID_AXES
    gmax = max(b * c, a * c, a * b)
    out = []
    need = n
    while need > 0:
        m = int(need * 1.6) + 64
        u = rng.standard_normal((m, 3))
        u /= np.linalg.norm(u, axis=1)[:, None]
        g = np.sqrt((b * c * u[:, 0]) ** 2 + (a * c * u[:, 1]) ** 2 + (a * b * u[:, 2]) ** 2)
        keep = rng.random(m) * gmax < g
        pts = u[keep] * np.array([a, b, c])
        out.append(pts[:need])
        need -= min(need, pts.shape[0])
    return np.concatenate(out)


def ellipsoid_plates(n: int, seed: int) -> np.ndarray:
    """Ellipsoid (5, 0.5, 0.5) plus two 4 x 1 plates at z = +-1.5, points
    split in proportion to area (BASELINE configs[2..4]; plate placement is
    not fixed by BASELINE -- this is the builder's choice, as in the 2D
    analog)."""
    rng = np.random.default_rng(seed)
    a_ell = spheroid_area(ELLIPSOID_AXES[0], ELLIPSOID_AXES[1])
    a_pl = PLATE_SIZE[0] * PLATE_SIZE[1]
    total = a_ell + 2.0 * a_pl
    n_e = int(round(n * a_ell / total))
    n_top = (n - n_e) // 2
    n_bot = n - n_e - n_top
    ell = _ellipsoid_surface(n_e, rng)

    def plate(m, z):
        xy = rng.random((m, 2)) * np.array(PLATE_SIZE) - 0.5 * np.array(PLATE_SIZE)
        return np.column_stack((xy, np.full(m, z)))

    return np.concatenate((ell, plate(n_top, PLATE_Z), plate(n_bot, -PLATE_Z)))


def surface_area(kind: str) -> float:
    if kind == "sphere":
        return 4.0 * math.pi
    if kind == "ellipsoid-plates":
        return spheroid_area(ELLIPSOID_AXES[0], ELLIPSOID_AXES[1]) + 2.0 * PLATE_SIZE[0] * PLATE_SIZE[1]
    raise ValueError(f"unknown surface {kind!r}")


def generate_surface(kind: str, n: int, seed: int) -> np.ndarray:
    if kind == "sphere":
        pts = sphere_surface(n, seed)
    elif kind == "ellipsoid-plates":
        pts = ellipsoid_plates(n, seed)
    else:
        raise ValueError(f"unknown surface {kind!r}")
    if np.unique(pts, axis=0).shape[0] != n:
        raise ValueError("generated coincident points; change n or seed")
    return pts


def wavenumber3(kind: str, n: int, points_per_wavelength: float = 10.0) -> float:
    """k = 2 pi / lambda, lambda = ppw * sqrt(area / n)."""
    h = math.sqrt(surface_area(kind) / n)
    return 2.0 * math.pi / (points_per_wavelength * h)


# ----------------------------------------------------------------------------
# kernel and auxiliary spheres (linalg.py restated)
# ----------------------------------------------------------------------------
def sphere_points(center, radius: float, count: int) -> np.ndarray:
    """count points on a sphere: Fibonacci lattice z_i = 1 - (2i + 1)/count,
    azimuth i * golden angle (the 3D counterpart of circle_points,
    linalg.py:70-81: deterministic, starts at the same place every call)."""
    if radius <= 0:
        raise ValueError("radius must be positive")
    if count < 3:
        raise ValueError("need at least 3 sphere points")
    i = np.arange(count)
    z = 1.0 - (2.0 * i + 1.0) / count
    r = np.sqrt(1.0 - z * z)
    phi = i * (math.pi * (3.0 - math.sqrt(5.0)))
    return np.column_stack((center[0] + radius * r * np.cos(phi),
                            center[1] + radius * r * np.sin(phi),
                            center[2] + radius * z))


def helmholtz_matrix(targets, sources, k: float, same_set: bool = False) -> np.ndarray:
    """G_ij = exp(-j k r_ij) / (4 pi r_ij), column-major (kernel_matrix,
    linalg.py:22-44: zero diagonal for a same set, coincident points are an
    error otherwise)."""
    t = np.asarray(targets, dtype=float)
    s = np.asarray(sources, dtype=float)
    diff = t[:, None, :] - s[None, :, :]
    d2 = np.einsum("ijk,ijk->ij", diff, diff)
    if same_set:
        np.fill_diagonal(d2, 1.0)
    elif (d2 == 0.0).any():
        raise ValueError("a target coincides with a source")
    r = np.sqrt(d2)
    g = np.exp(-1j * k * r) / (4.0 * math.pi * r)
    if same_set:
        np.fill_diagonal(g, 0.0)
    return np.asfortranarray(g)


def pinv(A: np.ndarray, rel_cutoff: float) -> np.ndarray:
    if not 0.0 < rel_cutoff < 1.0:
        raise ValueError("rel_cutoff must be in (0, 1)")
    return np.linalg.pinv(A, rcond=rel_cutoff)


# ----------------------------------------------------------------------------
# operators (operators.py restated)
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class HelmholtzParams:
    """operators.py:34-72 in 3D: ratios multiply the group half-side; k is
    the wavenumber.  The reference's validity rules with sqrt(3) (the cube's
    half-diagonal / h) in place of sqrt(2)."""

    Q: int = 24
    k: float = 1.0
    oversampling: int = 2
    rho_out_aux: float = 1.8
    rho_out_check: float = 2.15
    rho_in_check: float = 1.8
    rho_in_aux: float = 2.15
    pinv_cutoff: float = 1e-12

    def __post_init__(self):
        if self.Q < 3:
            raise ValueError("Q must be >= 3")
        if self.oversampling < 1:
            raise ValueError("oversampling must be >= 1")
        if not self.k >= 0.0:
            raise ValueError("k must be >= 0")
        if not SQRT3 < self.rho_out_aux < self.rho_out_check:
            raise ValueError("need sqrt(3) < rho_out_aux < rho_out_check")
        if not self.rho_in_check > SQRT3:
            raise ValueError("rho_in_check must exceed sqrt(3)")
        if not self.rho_in_aux > self.rho_in_check:
            raise ValueError("rho_in_aux must exceed rho_in_check")
        if not self.rho_out_check < 4.0 - self.rho_in_check:
            raise ValueError("rho_out_check too large for 4h separation")
        if not self.rho_out_aux + self.rho_in_check < 4.0:
            raise ValueError("rho_out_aux + rho_in_check must be < 4")

    @property
    def n_check(self) -> int:
        return self.oversampling * self.Q


@dataclass(frozen=True)
class GroupAux3:
    center: tuple
    half_side: float
    out_aux: np.ndarray
    out_check: np.ndarray
    in_aux: np.ndarray
    in_check: np.ndarray


def aux_at3(center, h: float, p: HelmholtzParams) -> GroupAux3:
    return GroupAux3(center=tuple(center), half_side=h,
                     out_aux=sphere_points(center, p.rho_out_aux * h, p.Q),
                     out_check=sphere_points(center, p.rho_out_check * h, p.n_check),
                     in_aux=sphere_points(center, p.rho_in_aux * h, p.Q),
                     in_check=sphere_points(center, p.rho_in_check * h, p.n_check))


def outgoing_fit3(aux: GroupAux3, p: HelmholtzParams) -> np.ndarray:
    return pinv(helmholtz_matrix(aux.out_check, aux.out_aux, p.k), p.pinv_cutoff)


def incoming_fit3(aux: GroupAux3, p: HelmholtzParams) -> np.ndarray:
    return pinv(helmholtz_matrix(aux.in_check, aux.in_aux, p.k), p.pinv_cutoff)


@dataclass
class HelmholtzOperatorSet:
    """All operators of one octree, keyed like OperatorSet (operators.py:158-174)."""

    params: HelmholtzParams
    V: dict = field(default_factory=dict)
    U: dict = field(default_factory=dict)
    C: dict = field(default_factory=dict)
    B: dict = field(default_factory=dict)
    D: dict = field(default_factory=dict)
    near: dict = field(default_factory=dict)


@dataclass
class HelmholtzTables:
    """Array form of the same operators (what the device plan consumes)."""

    params: HelmholtzParams
    C: np.ndarray            # (L - l0, 8, Q, Q) complex128, child level l0+1+i, octant
    B: np.ndarray
    D: np.ndarray            # (n_dtab, Q, Q) unique per (level, dx, dy, dz)
    d_index: np.ndarray      # (nnz,) per interaction entry
    octant: np.ndarray       # (G,) int32
    V: list                  # per leaf (Q, n_a) complex128
    U: list                  # per leaf (n_a, Q)


def _octants():
    return [(qx, qy, qz) for qx in (0, 1) for qy in (0, 1) for qz in (0, 1)]


def build_tables3(tree: Octree, p: HelmholtzParams) -> HelmholtzTables:
    """operators.py:177-253 in 3D: per-level fits, leaf V / U at the leaf's
    true center, C / B per (level, octant), D per (level, offset)."""
    a = tree.arrays
    side = tree.root_side
    Q = p.Q
    nl = tree.L - tree.l0
    ref_aux, out_fits, in_fits = {}, {}, {}
    for lv in range(tree.l0, tree.L + 1):
        h = side / (1 << (lv + 1))
        ref_aux[lv] = aux_at3((0.0, 0.0, 0.0), h, p)
        out_fits[lv] = outgoing_fit3(ref_aux[lv], p)
        in_fits[lv] = incoming_fit3(ref_aux[lv], p)
    C = np.zeros((max(nl, 0), 8, Q, Q), np.complex128)
    B = np.zeros_like(C)
    for lv in range(tree.l0 + 1, tree.L + 1):
        h = side / (1 << (lv + 1))
        parent = aux_at3((0.0, 0.0, 0.0), 2 * h, p)
        for o, (qx, qy, qz) in enumerate(_octants()):
            child = aux_at3(((2 * qx - 1) * h, (2 * qy - 1) * h, (2 * qz - 1) * h), h, p)
            C[lv - tree.l0 - 1, o] = out_fits[lv - 1] @ helmholtz_matrix(
                parent.out_check, child.out_aux, p.k)
            B[lv - tree.l0 - 1, o] = in_fits[lv] @ helmholtz_matrix(
                child.in_check, parent.in_aux, p.k)
    # translation: unique (level, dx, dy, dz)
    G = a.n_groups
    src_of = np.repeat(np.arange(G), np.diff(a.int_ptr))
    dst = a.int_idx
    off = a.ijk[dst] - a.ijk[src_of]
    lvl = a.level[src_of].astype(np.int64)
    keys = np.column_stack((lvl, off))
    uniq, d_index = np.unique(keys, axis=0, return_inverse=True)
    D = np.empty((uniq.shape[0], Q, Q), np.complex128)
    for j, (lv, dx, dy, dz) in enumerate(uniq.tolist()):
        h = side / (1 << (lv + 1))
        beta = aux_at3((2 * h * dx, 2 * h * dy, 2 * h * dz), h, p)
        D[j] = _translation(ref_aux[lv], beta, p, in_fits[lv])
    V, U = [], []
    ctr = a.center()
    hs = a.half_side()
    for g in range(a.level_count[tree.L]):
        aux = aux_at3(tuple(ctr[g]), float(hs[g]), p)
        pts = tree.points[a.start[g]:a.stop[g]]
        V.append(out_fits[tree.L] @ helmholtz_matrix(aux.out_check, pts, p.k))
        U.append(helmholtz_matrix(pts, aux.in_aux, p.k))
    return HelmholtzTables(params=p, C=C, B=B, D=D, d_index=d_index.ravel().astype(np.int64),
                           octant=a.octant(), V=V, U=U)


def _translation(alpha: GroupAux3, beta: GroupAux3, p: HelmholtzParams, fit) -> np.ndarray:
    dist = math.dist(alpha.center, beta.center)
    min_dist = (p.rho_out_aux + p.rho_in_check) * alpha.half_side
    if dist <= min_dist * (1.0 + 1e-12):
        raise ValueError("groups not well separated for translation")
    return fit @ helmholtz_matrix(alpha.in_check, beta.out_aux, p.k)


def near_block3(tree: Octree, a_id: int, b_id: int, k: float) -> np.ndarray:
    ar = tree.arrays
    pa = tree.points[ar.start[a_id]:ar.stop[a_id]]
    pb = tree.points[ar.start[b_id]:ar.stop[b_id]]
    return helmholtz_matrix(pa, pb, k, same_set=(a_id == b_id))


def build_all3(tree: Octree, p: HelmholtzParams,
               tables: HelmholtzTables | None = None) -> HelmholtzOperatorSet:
    """Dict form keyed like the reference's OperatorSet (operators.py:177-253):
    shared C / B / D objects per cache key, near blocks with the transposed
    partner shared (G is symmetric, so K_ba = K_ab^T)."""
    t = tables if tables is not None else build_tables3(tree, p)
    a = tree.arrays
    ops = HelmholtzOperatorSet(params=p)
    for g in range(a.level_count[tree.L]):
        ops.V[g] = t.V[g]
        ops.U[g] = t.U[g]
    # one object per cache key (operators.py:213-239 shares them the same way)
    Cv = {k: t.C[k] for k in np.ndindex(*t.C.shape[:2])}
    Bv = {k: t.B[k] for k in np.ndindex(*t.B.shape[:2])}
    Dv = [t.D[j] for j in range(t.D.shape[0])]
    for g in np.flatnonzero(a.parent >= 0).tolist():
        key = (int(a.level[g]) - tree.l0 - 1, int(t.octant[g]))
        ops.C[g] = Cv[key]
        ops.B[g] = Bv[key]
    ip, ii = a.int_ptr, a.int_idx
    for g in range(a.n_groups):
        for e in range(ip[g], ip[g + 1]):
            ops.D[(g, int(ii[e]))] = Dv[t.d_index[e]]
    for g in range(a.level_count[tree.L]):
        for nb in a.nbr_idx[a.nbr_ptr[g]:a.nbr_ptr[g + 1]].tolist():
            if nb < g:
                continue
            blk = near_block3(tree, g, nb, p.k)
            ops.near[(g, nb)] = blk
            if nb != g:
                ops.near[(nb, g)] = blk.T
    return ops


def dense_helmholtz(points: np.ndarray, q: np.ndarray, k: float, chunk: int = 512) -> np.ndarray:
    """phi_i = sum_{j != i} G(x_i, x_j) q_j (dense.py:14-33 with the
    Helmholtz kernel), O(N^2) in row chunks -- the accuracy reference."""
    pts = np.asarray(points, dtype=float)
    n = pts.shape[0]
    out = np.empty(np.shape(q), np.complex128)
    for s in range(0, n, chunk):
        e = min(s + chunk, n)
        diff = pts[s:e, None, :] - pts[None, :, :]
        r = np.sqrt(np.einsum("ijk,ijk->ij", diff, diff))
        idx = np.arange(s, e)
        r[idx - s, idx] = 1.0
        g = np.exp(-1j * k * r) / (4.0 * math.pi * r)
        g[idx - s, idx] = 0.0
        out[s:e] = g @ q
    return out


def track_b_problem(kind: str, n: int, seed: int, P: int, Q: int,
                    points_per_wavelength: float = 10.0):
    """(points, octree, params, q) for a BASELINE Track B configuration."""
    from .octree import build_octree
    pts = generate_surface(kind, n, seed)
    tree = build_octree(pts, TreeParams(P=P))
    params = HelmholtzParams(Q=Q, k=wavenumber3(kind, n, points_per_wavelength))
    rng = np.random.default_rng(seed)
    q = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return pts, tree, params, q
