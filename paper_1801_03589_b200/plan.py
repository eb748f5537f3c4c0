"""Plan exporter: Tree + operators -> device plan (libnesa_b200.so).

The reference keeps its operators as Python dicts of small numpy matrices
(operators.py:158-174) and walks them one gemv task at a time
(fastmvp.py:68-121).  A :class:`NesaPlan` flattens the same information into
the C ABI's descriptor (include/nesa_b200.h):

* tree arrays (perm, group ranges, parents, quadrants, level ranges, the
  neighbor and interaction CSR) -- straight from ``Tree.arrays``;
* the shared C / B (per level and quadrant) and unique D tables, with one D
  index per interaction entry;
* the per-leaf blocks: either taken from a host ``OperatorSet`` (drop-in for
  the reference's ``build_all`` output) or assembled on the device from the
  geometry (``assemble="device"``; no host near blocks at all).

The plan owns every device buffer; vectors are passed per call.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _capi
from .operators import NesaParams, OperatorSet, OperatorTables, build_tables
from .quadtree import Tree

_DTYPES = {"f64": _capi.NESA_F64, "float64": _capi.NESA_F64, "complex128": _capi.NESA_F64,
           "f32": _capi.NESA_F32, "float32": _capi.NESA_F32, "complex64": _capi.NESA_F32}


def _ptr(a: np.ndarray | None, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def _tables_from_opset(tree: Tree, ops: OperatorSet):
    """Recover C/B quadrant tables and a deduplicated D table from dicts."""
    a = tree.arrays
    Q = ops.params.Q
    nl = tree.L - tree.l0
    C = np.zeros((max(nl, 0), 4, Q, Q))
    B = np.zeros_like(C)
    seen = np.zeros((max(nl, 0), 4), bool)
    quad = (2 * (a.ix & 1) + (a.iy & 1)).astype(np.int32)
    for g in np.flatnonzero(a.parent >= 0).tolist():
        k = (int(a.level[g]) - tree.l0 - 1, int(quad[g]))
        if not seen[k]:
            C[k], B[k] = ops.C[g], ops.B[g]
            seen[k] = True
        elif not (np.array_equal(C[k], ops.C[g]) and np.array_equal(B[k], ops.B[g])):
            raise ValueError("C/B must be shared per (level, quadrant) as build_all makes them")
    ids = {}
    mats = []
    ip, ii = a.int_ptr, a.int_idx
    dindex = np.empty(ii.shape[0], np.int64)
    for g in range(a.n_groups):
        for e in range(ip[g], ip[g + 1]):
            m = ops.D[(g, int(ii[e]))]
            key = id(m)
            j = ids.get(key)
            if j is None:
                j = ids[key] = len(mats)
                mats.append(np.asarray(m, dtype=np.float64))
            dindex[e] = j
    D = np.stack(mats) if mats else np.zeros((0, Q, Q))
    return C, B, D, dindex, quad


def _blobs_from_opset(tree: Tree, ops: OperatorSet):
    a = tree.arrays
    nl = a.level_count[tree.L]
    near, V, U = [], [], []
    for g in range(nl):
        nb = a.nbr_idx[a.nbr_ptr[g]:a.nbr_ptr[g + 1]].tolist()
        slab = np.hstack([np.asarray(ops.near[(g, b)], dtype=np.float64) for b in nb])
        near.append(slab.ravel(order="F"))
        V.append(np.asarray(ops.V[g], dtype=np.float64).ravel(order="F"))
        U.append(np.asarray(ops.U[g], dtype=np.float64).ravel(order="F"))
    return np.concatenate(near), np.concatenate(V), np.concatenate(U)


def _radiation_blob(tree: Tree, tables: OperatorTables, leaf_range=None) -> np.ndarray:
    """Per-leaf V in the C ABI layout (Q x n column-major, leaves concatenated).

    Leaves outside ``leaf_range`` are left zero (the sub-plan never reads them).
    """
    from .operators import aux_at, build_radiation
    a = tree.arrays
    params = tables.params
    L = tree.L
    nl = a.level_count[L]
    lb, le = (0, nl) if leaf_range is None else leaf_range
    out = np.zeros(tree.n_points * params.Q)
    fit = tables.out_fit[L]
    for g in range(lb, le):
        s0, s1 = int(a.start[g]), int(a.stop[g])
        aux = aux_at(tuple(tables.leaf_center[g]), float(tables.leaf_h[g]), params)
        V = build_radiation(aux, tree.points[s0:s1], params, fit=fit)
        out[s0 * params.Q:s1 * params.Q] = V.ravel(order="F")
    return out


class NesaPlan:
    """Device plan of one (tree, operators, precision) triple.

    Parameters
    ----------
    tree : Tree
    ops : OperatorSet | OperatorTables | NesaParams
        ``OperatorSet`` (host matrices, e.g. from ``build_all`` -- reference's
        or ours) is uploaded as is; ``NesaParams`` / ``OperatorTables`` make
        the plan assemble near, V and U on the device.
    dtype : "f64" (float64 / complex128 vectors) or "f32" (float32 / complex64).
    device : CUDA device ordinal.
    leaf_range : (begin, end) leaf ids of this rank's targets (multi-GPU).
    stored_vu : keep stored V / U blocks even for a float32 plan from
        geometry; products of more than 4 real columns then run the far
        field as batched GEMMs over 128-column passes (many right-hand
        sides, C5).
    v_on_host : assemble the radiation blocks V = fit @ K(check, pts) on the
        host, per leaf, exactly as operators.py:107-112 does (default for
        float64 plans).  V goes through the ill-conditioned pinv fit, which
        amplifies 1-ulp differences between the device and numpy ``log`` to
        ~1e-12 at Q >= 32; the host route keeps float64 parity at ~1e-14.
        Near and U blocks are direct kernel entries and always assemble on
        the device.
    """

    def __init__(self, tree: Tree, ops, dtype: str = "f64", device: int = 0,
                 leaf_range: tuple[int, int] | None = None, v_on_host: bool | None = None,
                 comm=None, rank: int = 0, nranks: int = 1, exchange=None, far_only: bool = False,
                 stored_vu: bool = False):
        self.lib = _capi.load()
        if dtype not in _DTYPES:
            raise ValueError(f"unknown dtype {dtype!r}")
        self.tree = tree
        self.ops_in = ops      # what the plan was built from (MvpPipeline builds siblings)
        self.dtype = "f64" if _DTYPES[dtype] == _capi.NESA_F64 else "f32"
        self.device = int(device)
        if isinstance(ops, OperatorSet):
            params = ops.params
            C, B, D, dindex, quad = _tables_from_opset(tree, ops)
            near_b, V_b, U_b = _blobs_from_opset(tree, ops)
            tables = None
        else:
            tables = ops if isinstance(ops, OperatorTables) else build_tables(tree, ops)
            params = tables.params
            C, B, D, dindex, quad = tables.C, tables.B, tables.D, tables.d_index, tables.quad
            near_b = V_b = U_b = None
        self.params: NesaParams = params
        a = tree.arrays
        L, l0 = tree.L, tree.l0
        keep = {}

        def arr(name, x, dt):
            keep[name] = np.ascontiguousarray(x, dtype=dt)
            return keep[name]

        d = _capi.NesaPlanDesc()
        d.abi_version = _capi.NESA_ABI_VERSION
        d.op_dtype = _DTYPES[self.dtype]
        d.Q = params.Q
        d.n_check = params.n_check
        d.N = tree.n_points
        d.n_leaves = a.level_count[L]
        d.n_groups = a.n_groups
        d.l0, d.L = l0, L
        i64 = ctypes.c_int64
        d.perm = _ptr(arr("perm", tree.perm, np.int64), i64)
        d.group_start = _ptr(arr("start", a.start, np.int64), i64)
        d.group_stop = _ptr(arr("stop", a.stop, np.int64), i64)
        d.parent = _ptr(arr("parent", a.parent, np.int64), i64)
        d.quad = _ptr(arr("quad", quad, np.int32), ctypes.c_int32)
        d.level_first = _ptr(arr("lf", [a.level_first[lv] for lv in range(l0, L + 1)],
                                 np.int64), i64)
        d.level_count = _ptr(arr("lc", [a.level_count[lv] for lv in range(l0, L + 1)],
                                 np.int64), i64)
        d.nbr_ptr = _ptr(arr("np", a.nbr_ptr, np.int64), i64)
        d.nbr_idx = _ptr(arr("ni", a.nbr_idx, np.int64), i64)
        d.int_ptr = _ptr(arr("ip", a.int_ptr, np.int64), i64)
        d.int_idx = _ptr(arr("ii", a.int_idx, np.int64), i64)
        d.int_dtab = _ptr(arr("id", dindex, np.int64), i64)
        f64 = ctypes.c_double
        d.C = _ptr(arr("C", C, np.float64), f64)
        d.B = _ptr(arr("B", B, np.float64), f64)
        d.D = _ptr(arr("D", D, np.float64), f64)
        d.n_dtab = D.shape[0]
        if near_b is not None:
            d.near_blob = _ptr(arr("nearb", near_b, np.float64), f64)
            d.V_blob = _ptr(arr("Vb", V_b, np.float64), f64)
            d.U_blob = _ptr(arr("Ub", U_b, np.float64), f64)
        else:
            nl = a.level_count[L]
            if v_on_host is None:
                v_on_host = self.dtype == "f64"
            if v_on_host:
                d.V_blob = _ptr(arr("Vb", _radiation_blob(tree, tables, leaf_range),
                                    np.float64), f64)
            d.points_tree = _ptr(arr("pts", tree.points, np.float64), f64)
            d.leaf_center = _ptr(arr("ctr", tables.leaf_center, np.float64), f64)
            # radii exactly as circle_points receives them: rho * h (operators.py:86-94)
            d.leaf_r_check = _ptr(arr("rck", params.rho_out_check * tables.leaf_h, np.float64), f64)
            d.leaf_r_inaux = _ptr(arr("rax", params.rho_in_aux * tables.leaf_h, np.float64), f64)
            d.out_fit_leaf = _ptr(arr("fit", tables.out_fit[L], np.float64), f64)
            th_c = 2.0 * np.pi * np.arange(params.n_check) / params.n_check
            th_a = 2.0 * np.pi * np.arange(params.Q) / params.Q
            d.check_cos = _ptr(arr("cc", np.cos(th_c), np.float64), f64)
            d.check_sin = _ptr(arr("cs", np.sin(th_c), np.float64), f64)
            d.aux_cos = _ptr(arr("ac", np.cos(th_a), np.float64), f64)
            d.aux_sin = _ptr(arr("as", np.sin(th_a), np.float64), f64)
            assert tables.leaf_h.shape[0] == nl
        if leaf_range is not None:
            d.leaf_begin, d.leaf_end = int(leaf_range[0]), int(leaf_range[1])
        # far_only: no near operator (extra plans of a many-RHS product)
        d.options = (_capi.NESA_PLAN_FAR_ONLY if far_only else 0) | \
            (_capi.NESA_PLAN_STORED_VU if stored_vu else 0)
        self.far_only = far_only
        self.stored_vu = stored_vu
        self.leaf_range = leaf_range
        h = ctypes.c_void_p()
        if comm is None:
            _capi.check(self.lib.nesa_plan_create(ctypes.byref(d), self.device, ctypes.byref(h)))
        else:
            # distributed plan: the halo exchange (pack -> ncclAllGather ->
            # combine) is captured into the product graph (nesa_plan_create_dist)
            xp = exchange
            x = _capi.NesaExchangeDesc()
            x.n_export = int(xp.export_ids.size)
            x.export_ids = _ptr(arr("xe", xp.export_ids, np.int64), i64)
            x.max_export = int(xp.max_export)
            x.n_import = int(xp.import_ids.size)
            x.import_ids = _ptr(arr("xi", xp.import_ids, np.int64), i64)
            x.max_contrib = int(xp.contrib.shape[1]) if xp.contrib.ndim == 2 else 1
            x.contrib = _ptr(arr("xc", xp.contrib.reshape(-1), np.int64), i64)
            _capi.check(self.lib.nesa_plan_create_dist(ctypes.byref(d), self.device, ctypes.c_void_p(comm),
                                                       int(rank), int(nranks), ctypes.byref(x),
                                                       ctypes.byref(h)))
        self._h = h
        self.n_dtab = int(D.shape[0])

    # ------------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            self.lib.nesa_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> ctypes.c_void_p:
        if not self._h.value:
            raise ValueError("plan is closed")
        return self._h

    def stat(self, name: str) -> int:
        return int(self.lib.nesa_plan_stat(self.handle, _capi.STAT[name]))

    @property
    def vec_dtype_real(self):
        return np.float64 if self.dtype == "f64" else np.float32

    def matvec_ptr(self, q_ptr: int, phi_ptr: int, nrhs: int, is_complex: bool,
                   near: bool = True, far: bool = True, stream: int = 0,
                   profile=False, stage: int = 0) -> None:
        """Raw device-pointer product (the C ABI call, stream-ordered).

        ``profile``: True records every stage's events; "near" only the
        near-field kernel's (no event nodes on the critical path).
        """
        flags = (_capi.NESA_NEAR if near else 0) | (_capi.NESA_FAR if far else 0)
        if profile:
            flags |= _capi.NESA_PROFILE
            if profile == "near":
                flags |= _capi.NESA_PROFILE_NEAR
        if stage == 0:
            rc = self.lib.nesa_matvec(self.handle, ctypes.c_void_p(q_ptr),
                                      ctypes.c_void_p(phi_ptr), nrhs, int(is_complex),
                                      flags, ctypes.c_void_p(stream))
        else:
            rc = self.lib.nesa_matvec_stage(self.handle, stage, ctypes.c_void_p(q_ptr),
                                            ctypes.c_void_p(phi_ptr), nrhs, int(is_complex),
                                            flags, ctypes.c_void_p(stream))
        _capi.check(rc)

    def matvec_cols_ptr(self, q_ptr: int, phi_ptr: int, ld_real: int, col0: int, ncols: int,
                        near: bool = True, far: bool = True, stream: int = 0) -> None:
        """Columns [col0, col0 + ncols) of (N, ld_real) real device blocks."""
        flags = (_capi.NESA_NEAR if near else 0) | (_capi.NESA_FAR if far else 0)
        _capi.check(self.lib.nesa_matvec_cols(self.handle, ctypes.c_void_p(q_ptr),
                                              ctypes.c_void_p(phi_ptr), ld_real, col0, ncols, flags,
                                              ctypes.c_void_p(stream)))

    def near_wide_ptr(self, q_ptr: int, phi_ptr: int, ld_real: int, col0: int, ncols: int,
                      stream: int = 0) -> None:
        """phi[:, col0:col0+ncols] += near field of q (float32 + tensor cores,
        128 real columns per tcgen05 pass; operator streamed once)."""
        _capi.check(self.lib.nesa_matvec_near_wide(self.handle, ctypes.c_void_p(q_ptr),
                                                   ctypes.c_void_p(phi_ptr), ld_real, col0, ncols,
                                                   ctypes.c_void_p(stream)))

    def s_dev_ptr(self, nrhs_real: int) -> int:
        p = self.lib.nesa_plan_s_dev(self.handle, nrhs_real)
        if not p:
            raise RuntimeError(self.lib.nesa_last_error().decode())
        return int(p)

    def profile_reset(self) -> None:
        _capi.check(self.lib.nesa_profile_reset(self.handle))

    def profile_read(self, stage: str, max_n: int = 100000) -> np.ndarray:
        buf = (ctypes.c_float * max_n)()
        n = self.lib.nesa_profile_read(self.handle, _capi.STAGE[stage], buf, max_n)
        if n < 0:
            raise RuntimeError(self.lib.nesa_last_error().decode())
        return np.frombuffer(buf, dtype=np.float32, count=n).astype(np.float64)

    def trace_read(self, max_n: int = 64) -> list[tuple[str, float]]:
        """(kernel, ms from the product start) after each kernel of the last
        profiled product; needs NESA_TRACE=1 when the plan was created."""
        buf = (ctypes.c_float * max_n)()
        n = self.lib.nesa_trace_read(self.handle, buf, max_n)
        if n < 0:
            raise RuntimeError(self.lib.nesa_last_error().decode())
        return [(self.lib.nesa_trace_name(self.handle, i).decode(), float(buf[i])) for i in range(n)]


def algorithmic_bytes(plan: NesaPlan, nrhs_real: int, near: bool = True,
                      far: bool = True) -> dict:
    """B_alg of SURVEY.md §8d for one product, split by kernel.

    s_m = operator entry bytes, s_v = real vector element bytes.
    near: E_near * s_m + (gathered x + written y) vectors;
    V/U:  N*Q * s_m each plus their vectors; C/B/D: unique tables once.
    """
    sm = 8 if plan.dtype == "f64" else 4
    sv = sm * nrhs_real
    t = plan.tree
    N = t.n_points
    G = t.arrays.n_groups
    Q = plan.params.Q
    e_near = plan.stat("near_entries")
    out = {}
    out["near"] = e_near * sm + 2 * N * sv if near else 0
    if far:
        out["radiation"] = plan.stat("v_entries") * sm + N * sv + G * Q * sv
        out["reception"] = plan.stat("u_entries") * sm + G * Q * sv + 2 * N * sv
        n_cb = 2 * 4 * max(t.L - t.l0, 0)
        out["transfer_tables"] = (n_cb + plan.n_dtab) * Q * Q * sm + 2 * G * Q * sv
    out["perm"] = 8 * N * 2
    out["vectors"] = 2 * N * sv
    out["total"] = (e_near * sm if near else 0) + (
        (plan.stat("v_entries") + plan.stat("u_entries")) * sm if far else 0) + \
        ((2 * 4 * max(t.L - t.l0, 0) + plan.n_dtab) * Q * Q * sm if far else 0) + \
        2 * N * sv + (4 * G * Q * sv if far else 0) + 8 * N
    return out


def algorithmic_flops(plan: NesaPlan, nrhs_real: int) -> float:
    """F of SURVEY.md §8d: 2*(E_near + 2NQ + (2(G-N_l0) + D_refs) Q^2) per column."""
    t = plan.tree
    Q = plan.params.Q
    n_l0 = t.arrays.level_count[t.l0]
    G = t.arrays.n_groups
    return 2.0 * nrhs_real * (plan.stat("near_entries") + plan.stat("v_entries") +
                              plan.stat("u_entries") +
                              (2 * (G - n_l0) + plan.stat("d_refs")) * Q * Q)


def log2ceil(x: int) -> int:
    return int(math.ceil(math.log2(max(x, 1))))
