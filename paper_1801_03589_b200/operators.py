"""Equivalent-source operator assembly (host side).

Restates /root/reference/pkg/src/taskfmm/operators.py:34-253.  Each group
carries an outgoing and an incoming circle of Q auxiliary sources; V, C, D,
B, U are fitted through a truncated-SVD pinv on oversampled check circles.
Scale invariance makes C/B one matrix per (level, child quadrant) and D one
per (level, integer offset).

Two products:

* :func:`build_all` -> :class:`OperatorSet`, the reference's dict-of-matrices
  form (drop-in; the oracle and the host plan exporter read it).
* :func:`build_tables` -> :class:`OperatorTables`, the compact form the GPU
  plan is made of: per-level fits, the C/B quadrant tables, the unique D
  table with one index per interaction-list entry, and the per-leaf aux
  circle geometry so V, U and the near blocks can be assembled on device
  (csrc/nesa_assemble.cu) instead of on the host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .linalg import DEFAULT_PINV_CUTOFF, circle_points, kernel_matrix, pinv
from .quadtree import Group, Tree

SQRT2 = math.sqrt(2.0)


@dataclass(frozen=True)
class NesaParams:
    """Aux geometry; radii are multiples of the half side (operators.py:34-67)."""

    Q: int = 10
    oversampling: int = 2
    rho_out_aux: float = 1.45
    rho_out_check: float = 2.5
    rho_in_check: float = 1.45
    rho_in_aux: float = 2.8
    pinv_cutoff: float = DEFAULT_PINV_CUTOFF

    def __post_init__(self):
        if self.Q < 3:
            raise ValueError("Q must be >= 3")
        if self.oversampling < 1:
            raise ValueError("oversampling must be >= 1")
        if not SQRT2 < self.rho_out_aux < self.rho_out_check:
            raise ValueError("need sqrt(2) < rho_out_aux < rho_out_check")
        if not self.rho_in_check > SQRT2:
            raise ValueError("rho_in_check must exceed sqrt(2)")
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
class GroupAux:
    """Aux point sets of one group (operators.py:70-79)."""

    center: tuple[float, float]
    half_side: float
    out_aux: np.ndarray
    out_check: np.ndarray
    in_aux: np.ndarray
    in_check: np.ndarray


def aux_at(center, h: float, params: NesaParams) -> GroupAux:
    """The four circles of a group with center ``center`` and half side h."""
    return GroupAux(
        center=(center[0], center[1]), half_side=h,
        out_aux=circle_points(center, params.rho_out_aux * h, params.Q),
        out_check=circle_points(center, params.rho_out_check * h, params.n_check),
        in_aux=circle_points(center, params.rho_in_aux * h, params.Q),
        in_check=circle_points(center, params.rho_in_check * h, params.n_check))


def build_group_aux(g: Group, params: NesaParams) -> GroupAux:
    return aux_at(g.center, g.half_side, params)


def outgoing_fit(aux: GroupAux, params: NesaParams) -> np.ndarray:
    """pinv(K(out_check, out_aux)), shared by the V and C fits."""
    return pinv(kernel_matrix(aux.out_check, aux.out_aux), params.pinv_cutoff)


def incoming_fit(aux: GroupAux, params: NesaParams) -> np.ndarray:
    """pinv(K(in_check, in_aux)), shared by the D and B fits."""
    return pinv(kernel_matrix(aux.in_check, aux.in_aux), params.pinv_cutoff)


def build_radiation(aux, points, params, fit=None):
    """V (Q x n): leaf charges -> outgoing sources (operators.py:107-112)."""
    fit = outgoing_fit(aux, params) if fit is None else fit
    return fit @ kernel_matrix(aux.out_check, points)


def build_source_transfer(parent_aux, child_aux, params, fit=None):
    """C (Q x Q): child outgoing -> parent outgoing (operators.py:115-121)."""
    fit = outgoing_fit(parent_aux, params) if fit is None else fit
    return fit @ kernel_matrix(parent_aux.out_check, child_aux.out_aux)


def build_translation(alpha_aux, beta_aux, params, fit=None):
    """D (Q x Q): far outgoing -> incoming of alpha (operators.py:124-135)."""
    dist = math.hypot(alpha_aux.center[0] - beta_aux.center[0],
                      alpha_aux.center[1] - beta_aux.center[1])
    min_dist = (params.rho_out_aux + params.rho_in_check) * alpha_aux.half_side
    if dist <= min_dist * (1.0 + 1e-12):
        raise ValueError("groups not well separated for translation")
    fit = incoming_fit(alpha_aux, params) if fit is None else fit
    return fit @ kernel_matrix(alpha_aux.in_check, beta_aux.out_aux)


def build_potential_transfer(child_aux, parent_aux, params, fit=None):
    """B (Q x Q): parent incoming -> child incoming (operators.py:138-144)."""
    fit = incoming_fit(child_aux, params) if fit is None else fit
    return fit @ kernel_matrix(child_aux.in_check, parent_aux.in_aux)


def build_reception(aux, points):
    """U (n x Q): incoming sources -> potentials at the points."""
    return kernel_matrix(points, aux.in_aux)


def build_near_block(points_a, points_b, same: bool):
    """Dense kernel block of two touching leaves; zero diagonal if same."""
    return kernel_matrix(points_a, points_b, same_set=same)


@dataclass
class OperatorSet:
    """Operators keyed by group id / id pair (operators.py:158-174)."""

    params: NesaParams
    V: dict = field(default_factory=dict)
    U: dict = field(default_factory=dict)
    C: dict = field(default_factory=dict)
    B: dict = field(default_factory=dict)
    D: dict = field(default_factory=dict)
    near: dict = field(default_factory=dict)

    def entry_count(self) -> int:
        return sum(m.size for t in (self.V, self.U, self.C, self.B, self.D, self.near)
                   for m in t.values())


# --------------------------------------------------------------------------
# Compact tables
# --------------------------------------------------------------------------

@dataclass
class OperatorTables:
    """Everything except the per-leaf/per-pair blocks, in array form.

    ``C[l - l0 - 1, 2*qx + qy]`` / ``B[...]`` are the transfer matrices for
    children at level l; ``D[d_index[e]]`` is the translation matrix of
    interaction entry e (aligned with ``tree.arrays.int_idx``).
    """

    params: NesaParams
    out_fit: dict            # level -> (Q, n_check)
    in_fit: dict
    C: np.ndarray            # (L - l0, 4, Q, Q)
    B: np.ndarray
    D: np.ndarray            # (nD, Q, Q)
    d_keys: np.ndarray       # (nD, 3) (level, dx, dy)
    d_index: np.ndarray      # (n_interaction_entries,) int64
    quad: np.ndarray         # (G,) child quadrant 2*(ix&1)+(iy&1)
    leaf_center: np.ndarray  # (NL, 2)
    leaf_h: np.ndarray       # (NL,)


def _level_fits(tree: Tree, params: NesaParams):
    side = tree.root_side
    ref_aux, out_fit, in_fit = {}, {}, {}
    for lv in range(tree.l0, tree.L + 1):
        h = side / (1 << (lv + 1))
        ref_aux[lv] = aux_at((0.0, 0.0), h, params)
        out_fit[lv] = outgoing_fit(ref_aux[lv], params)
        in_fit[lv] = incoming_fit(ref_aux[lv], params)
    return ref_aux, out_fit, in_fit


def _transfer_tables(tree: Tree, params: NesaParams, out_fit, in_fit):
    """C/B per (level, quadrant) (operators.py:204-223)."""
    Q = params.Q
    nl = tree.L - tree.l0
    C = np.zeros((nl, 4, Q, Q))
    B = np.zeros((nl, 4, Q, Q))
    side = tree.root_side
    for lv in range(tree.l0 + 1, tree.L + 1):
        h = side / (1 << (lv + 1))
        parent = aux_at((0.0, 0.0), 2 * h, params)
        for qx in (0, 1):
            for qy in (0, 1):
                child = aux_at(((2 * qx - 1) * h, (2 * qy - 1) * h), h, params)
                C[lv - tree.l0 - 1, 2 * qx + qy] = build_source_transfer(
                    parent, child, params, fit=out_fit[lv - 1])
                B[lv - tree.l0 - 1, 2 * qx + qy] = build_potential_transfer(
                    child, parent, params, fit=in_fit[lv])
    return C, B


def _translation_tables(tree: Tree, params: NesaParams, ref_aux, in_fit):
    """Unique D per (level, dx, dy) plus the per-entry index (operators.py:225-239)."""
    a = tree.arrays
    src = np.repeat(np.arange(a.n_groups), np.diff(a.int_ptr))
    dst = a.int_idx
    lvl = a.level[src].astype(np.int64)
    dx = a.ix[dst] - a.ix[src]
    dy = a.iy[dst] - a.iy[src]
    keys = np.stack((lvl, dx, dy), axis=1)
    if keys.shape[0] == 0:
        return (np.zeros((0, params.Q, params.Q)), np.zeros((0, 3), np.int64),
                np.zeros(0, np.int64))
    uk, inv = np.unique(keys, axis=0, return_inverse=True)
    side = tree.root_side
    D = np.empty((uk.shape[0], params.Q, params.Q))
    for i, (lv, ddx, ddy) in enumerate(uk.tolist()):
        h = side / (1 << (lv + 1))
        beta = aux_at((2 * h * ddx, 2 * h * ddy), h, params)
        D[i] = build_translation(ref_aux[lv], beta, params, fit=in_fit[lv])
    return D, uk, inv.reshape(-1).astype(np.int64)


def build_tables(tree: Tree, params: NesaParams) -> OperatorTables:
    """Compact operator tables for the device plan (no per-leaf blocks)."""
    ref_aux, out_fit, in_fit = _level_fits(tree, params)
    C, B = _transfer_tables(tree, params, out_fit, in_fit)
    D, d_keys, d_index = _translation_tables(tree, params, ref_aux, in_fit)
    a = tree.arrays
    quad = (2 * (a.ix & 1) + (a.iy & 1)).astype(np.int32)
    nl = a.level_count[tree.L]
    return OperatorTables(params=params, out_fit=out_fit, in_fit=in_fit, C=C, B=B,
                          D=D, d_keys=d_keys, d_index=d_index, quad=quad,
                          leaf_center=a.center()[:nl], leaf_h=a.half_side()[:nl])


def build_all(tree: Tree, params: NesaParams) -> OperatorSet:
    """The complete reference-format operator set (operators.py:177-253)."""
    ops = OperatorSet(params=params)
    t = build_tables(tree, params)
    a = tree.arrays
    L, l0 = tree.L, tree.l0
    nl = a.level_count[L]
    for g in range(nl):
        aux = aux_at(tuple(t.leaf_center[g]), float(t.leaf_h[g]), params)
        pts = tree.points[a.start[g]:a.stop[g]]
        ops.V[g] = build_radiation(aux, pts, params, fit=t.out_fit[L])
        ops.U[g] = build_reception(aux, pts)
    for g in np.flatnonzero(a.parent >= 0).tolist():
        k = (int(a.level[g]) - l0 - 1, int(t.quad[g]))
        ops.C[g] = t.C[k]
        ops.B[g] = t.B[k]
    views = [t.D[i] for i in range(t.D.shape[0])]     # shared, like d_cache
    ip, ii = a.int_ptr, a.int_idx
    for g in range(a.n_groups):
        for e in range(ip[g], ip[g + 1]):
            ops.D[(g, int(ii[e]))] = views[t.d_index[e]]
    np_, ni = a.nbr_ptr, a.nbr_idx
    for g in range(nl):
        pa = tree.points[a.start[g]:a.stop[g]]
        for nid in ni[np_[g]:np_[g + 1]].tolist():
            if nid < g:
                continue
            blk = build_near_block(pa, tree.points[a.start[nid]:a.stop[nid]],
                                   same=(nid == g))
            ops.near[(g, nid)] = blk
            if nid != g:
                ops.near[(nid, g)] = blk.T
    return ops
