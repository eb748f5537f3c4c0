"""Bounded CPU-baseline sample of the reference path -- TEST/BENCH INFRASTRUCTURE.

bench.py's ``cpu_baseline`` leg and ``--impl reference`` time the oracle
(oracle/mvp_oracle.mvp_serial, the restated reference loop) on the first
``fraction`` of every stage loop of one product, so a step stays ~0.1-1 s at
N = 2M.  Only the operators those iterations touch are assembled (the
reference's build_all at 2M takes ~35 s and 6 GB); they come
from the host assembly that tests/test_oracle.py pins to the reference's
checksums.
"""

from __future__ import annotations

import math
import time

import numpy as np

from paper_1801_03589_b200.operators import (OperatorSet, aux_at, build_near_block,
                                             build_radiation, build_reception, build_tables)

from .mvp_oracle import mvp_serial


def build_sampled_opset(tree, params, fraction: float) -> OperatorSet:
    """OperatorSet holding every operator the sampled loops of mvp_serial use."""
    t = build_tables(tree, params)
    a = tree.arrays
    L, l0 = tree.L, tree.l0
    ops = OperatorSet(params=params)
    nl = a.level_count[L]
    n_s = int(math.ceil(fraction * nl))
    for g in range(n_s):
        aux = aux_at(tuple(t.leaf_center[g]), float(t.leaf_h[g]), params)
        pts = tree.points[a.start[g]:a.stop[g]]
        ops.V[g] = build_radiation(aux, pts, params, fit=t.out_fit[L])
        ops.U[g] = build_reception(aux, pts)
        for nid in a.nbr_idx[a.nbr_ptr[g]:a.nbr_ptr[g + 1]].tolist():
            ops.near[(g, nid)] = build_near_block(
                pts, tree.points[a.start[nid]:a.stop[nid]], same=(nid == g))
    for g in np.flatnonzero(a.parent >= 0).tolist():
        k = (int(a.level[g]) - l0 - 1, int(t.quad[g]))
        ops.C[g] = t.C[k]
        ops.B[g] = t.B[k]
    views = [t.D[i] for i in range(t.D.shape[0])]
    ip, ii = a.int_ptr, a.int_idx
    for g in range(a.n_groups):
        for e in range(ip[g], ip[g + 1]):
            ops.D[(g, int(ii[e]))] = views[t.d_index[e]]
    return ops


def time_sample(tree, ops, q: np.ndarray, fraction: float) -> float:
    """Seconds of one sampled complex product, as the reference runs it:
    two real mvp_serial calls (Re, Im), summed."""
    t = 0.0
    parts = (q.real.astype(np.float64), q.imag.astype(np.float64)) if np.iscomplexobj(q) \
        else (q.astype(np.float64),)
    for part in parts:
        t0 = time.perf_counter()
        mvp_serial(tree, ops, part, fraction=fraction)
        t += time.perf_counter() - t0
    return t
