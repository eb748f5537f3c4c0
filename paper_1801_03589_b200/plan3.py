"""Track B device plan: octree + complex (Helmholtz) operators on the same engine.

The engine (csrc/nesa_plan.cu) multiplies real operators into vectors of
R interleaved real columns.  A complex operator M = A + iB enters in its
real embedding: every entry a + ib becomes the 2 x 2 block [[a, -b], [b, a]]
acting on the (re, im) pair of one complex unknown.  Laid out that way a
complex vector of N entries is, byte for byte, a real vector of 2N entries,
so the plan sees a "tree" whose point ranges, Q and N are doubled and runs
the product with one real column -- the radiation / reception blocks and
the C / D / B transfers all do complex arithmetic (4 real multiply-adds per
complex one, exactly the complex flop count) with no new kernel.  The near
field, which streams the dominant operator bytes, does not pay the
embedding's 2x storage: its blob is row-split (rows Re / Im of each complex
row, NESA_PLAN_COMPLEX_NEAR) and the near kernel's complex-store epilogue
(kModeStoreCplx) combines each row pair, so it reads 8 bytes per complex
float32 entry; the radiation V and reception U blocks are row-split the same
way (kModeScatterCplx scatters the reception's complex rows).  NESA_PLAN_OCTREE tells the plan that the tree has 8 child
kinds (octants) per level and that its operators come from the host.

Reference anchor: the product is fastmvp.py:142-172 on the operators of
helmholtz.build_tables3 (operators.py:177-253 restated in 3D); its checker
is oracle/mvp_oracle.mvp_serial (dtype-generic) on build_all3's dicts.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _capi
from .helmholtz import HelmholtzOperatorSet, HelmholtzParams, HelmholtzTables, build_tables3, near_block3
from .octree import Octree
from .plan import NesaPlan, _DTYPES, _ptr


def embed(M: np.ndarray) -> np.ndarray:
    """Complex (..., m, n) -> real (..., 2m, 2n) with 2x2 blocks [[a, -b], [b, a]]."""
    M = np.asarray(M)
    m, n = M.shape[-2:]
    R = np.empty(M.shape[:-2] + (2 * m, 2 * n), np.float64)
    R[..., 0::2, 0::2] = M.real
    R[..., 0::2, 1::2] = -M.imag
    R[..., 1::2, 0::2] = M.imag
    R[..., 1::2, 1::2] = M.real
    return R


def row_split(M: np.ndarray) -> np.ndarray:
    """Complex (m, n) -> real (2m, n): row 2r = Re M[r], row 2r+1 = Im M[r]."""
    M = np.asarray(M)
    R = np.empty((2 * M.shape[0], M.shape[1]), np.float64)
    R[0::2] = M.real
    R[1::2] = M.imag
    return R


def _tables_from_opset3(tree: Octree, ops: HelmholtzOperatorSet):
    """Recover the per-(level, octant) C / B and a deduplicated D table from
    build_all3's dicts (shared objects per cache key, like operators.py)."""
    a = tree.arrays
    Q = ops.params.Q
    nl = tree.L - tree.l0
    octant = a.octant()
    C = np.zeros((max(nl, 0), 8, Q, Q), np.complex128)
    B = np.zeros_like(C)
    for g in np.flatnonzero(a.parent >= 0).tolist():
        k = (int(a.level[g]) - tree.l0 - 1, int(octant[g]))
        C[k], B[k] = ops.C[g], ops.B[g]
    ids, mats = {}, []
    dindex = np.empty(a.int_idx.shape[0], np.int64)
    for g in range(a.n_groups):
        for e in range(a.int_ptr[g], a.int_ptr[g + 1]):
            m = ops.D[(g, int(a.int_idx[e]))]
            j = ids.get(id(m))
            if j is None:
                j = ids[id(m)] = len(mats)
                mats.append(np.asarray(m, np.complex128))
            dindex[e] = j
    D = np.stack(mats) if mats else np.zeros((0, Q, Q), np.complex128)
    return C, B, D, dindex, octant


class HelmholtzPlan(NesaPlan):
    """Device plan of one (octree, Helmholtz operators, precision) triple.

    ops: HelmholtzParams (tables built here), HelmholtzTables, or a
    HelmholtzOperatorSet (build_all3 dicts, uploaded as they are).  From
    params / tables the near blocks are evaluated on the device
    (NESA_PLAN_HELMHOLTZ_NEAR); V / U (through the pinv fits) come from the
    host.
    dtype: "c128" (float64 engine) or "c64" (float32 engine).
    """

    def __init__(self, tree: Octree, ops, dtype: str = "c128", device: int = 0,
                 complex_near: bool = True):
        self.lib = _capi.load()
        dt = {"c128": "f64", "complex128": "f64", "f64": "f64",
              "c64": "f32", "complex64": "f32", "f32": "f32"}.get(dtype)
        if dt is None:
            raise ValueError(f"unknown dtype {dtype!r}")
        self.tree = tree
        self.ops_in = ops
        self.dtype = dt
        self.device = int(device)
        self.far_only = False
        self.leaf_range = None
        a = tree.arrays
        L, l0 = tree.L, tree.l0
        nl = a.level_count[L]
        if isinstance(ops, HelmholtzOperatorSet):
            params = ops.params
            C, B, D, dindex, octant = _tables_from_opset3(tree, ops)
            V = [ops.V[g] for g in range(nl)]
            U = [ops.U[g] for g in range(nl)]
            near_of = lambda g, b: ops.near[(g, b)]  # noqa: E731
        else:
            t: HelmholtzTables = ops if isinstance(ops, HelmholtzTables) else build_tables3(tree, ops)
            params = t.params
            C, B, D, dindex, octant = t.C, t.B, t.D, t.d_index, t.octant
            V, U = t.V, t.U
            near_of = None   # assembled on the device (NESA_PLAN_HELMHOLTZ_NEAR)
        self.params: HelmholtzParams = params
        Q = params.Q
        if near_of is None and not complex_near:
            near_of = lambda g, b: near_block3(tree, g, b, params.k)  # noqa: E731
        near, Vb, Ub = [], [], []
        for g in range(nl):
            if near_of is not None:
                nb = a.nbr_idx[a.nbr_ptr[g]:a.nbr_ptr[g + 1]].tolist()
                slab = np.hstack([near_of(g, b) for b in nb])
                near.append((row_split(slab) if complex_near else embed(slab)).ravel(order="F"))
            Vb.append((row_split(V[g]) if complex_near else embed(V[g])).ravel(order="F"))
            Ub.append((row_split(U[g]) if complex_near else embed(U[g])).ravel(order="F"))
        keep = {}

        def arr(name, x, dtype_):
            keep[name] = np.ascontiguousarray(x, dtype=dtype_)
            return keep[name]

        i64, f64 = ctypes.c_int64, ctypes.c_double
        d = _capi.NesaPlanDesc()
        d.abi_version = _capi.NESA_ABI_VERSION
        d.op_dtype = _DTYPES[self.dtype]
        d.Q = 2 * Q
        d.n_check = 2 * params.n_check
        d.N = 2 * tree.n_points
        d.n_leaves = nl
        d.n_groups = a.n_groups
        d.l0, d.L = l0, L
        perm2 = (2 * tree.perm[:, None] + np.arange(2)[None, :]).reshape(-1)
        d.perm = _ptr(arr("perm", perm2, np.int64), i64)
        d.group_start = _ptr(arr("start", 2 * a.start, np.int64), i64)
        d.group_stop = _ptr(arr("stop", 2 * a.stop, np.int64), i64)
        d.parent = _ptr(arr("parent", a.parent, np.int64), i64)
        d.quad = _ptr(arr("quad", octant, np.int32), ctypes.c_int32)
        d.level_first = _ptr(arr("lf", [a.level_first[lv] for lv in range(l0, L + 1)], np.int64), i64)
        d.level_count = _ptr(arr("lc", [a.level_count[lv] for lv in range(l0, L + 1)], np.int64), i64)
        d.nbr_ptr = _ptr(arr("np", a.nbr_ptr, np.int64), i64)
        d.nbr_idx = _ptr(arr("ni", a.nbr_idx, np.int64), i64)
        d.int_ptr = _ptr(arr("ip", a.int_ptr, np.int64), i64)
        d.int_idx = _ptr(arr("ii", a.int_idx, np.int64), i64)
        d.int_dtab = _ptr(arr("id", dindex, np.int64), i64)
        d.C = _ptr(arr("C", embed(C.reshape(-1, Q, Q)) if C.size else np.zeros(1), np.float64), f64)
        d.B = _ptr(arr("B", embed(B.reshape(-1, Q, Q)) if B.size else np.zeros(1), np.float64), f64)
        d.D = _ptr(arr("D", embed(D) if D.size else np.zeros(1), np.float64), f64)
        d.n_dtab = D.shape[0]
        if near:
            d.near_blob = _ptr(arr("near", np.concatenate(near), np.float64), f64)
        else:
            # near blocks evaluated on the device from the 3D points
            d.points3 = _ptr(arr("pts3", tree.points, np.float64), f64)
            d.wavenumber = float(params.k)
        d.V_blob = _ptr(arr("V", np.concatenate(Vb), np.float64), f64)
        d.U_blob = _ptr(arr("U", np.concatenate(Ub), np.float64), f64)
        d.options = _capi.NESA_PLAN_OCTREE | (_capi.NESA_PLAN_COMPLEX_NEAR if complex_near else 0) | \
            (0 if near else _capi.NESA_PLAN_HELMHOLTZ_NEAR)
        self.complex_near = complex_near
        h = ctypes.c_void_p()
        _capi.check(self.lib.nesa_plan_create(ctypes.byref(d), self.device, ctypes.byref(h)))
        self._h = h
        self.n_dtab = int(D.shape[0])

    @property
    def complex_dtype(self):
        return np.complex128 if self.dtype == "f64" else np.complex64

    def matvec(self, q, near: bool = True, far: bool = True):
        """phi = K~ q for complex q of shape (N,) or (N, m), numpy or CUDA torch.

        Original point order in and out, like mvp (fastmvp.py:142-172)."""
        import torch
        n = self.tree.n_points
        is_np = isinstance(q, np.ndarray)
        cdt = torch.complex128 if self.dtype == "f64" else torch.complex64
        if is_np:
            qa = np.asarray(q)
            if qa.ndim not in (1, 2) or qa.shape[0] != n:
                raise ValueError("q must have one value per point")
            qt = torch.from_numpy(np.ascontiguousarray(qa, dtype=self.complex_dtype)).cuda(self.device)
        else:
            if q.dim() not in (1, 2) or q.shape[0] != n:
                raise ValueError("q must have one value per point")
            qt = q.to(device=f"cuda:{self.device}", dtype=cdt).contiguous()
        m = 1 if qt.dim() == 1 else qt.shape[1]
        # (N, m) complex = (N, m, 2) real; the embedded vector is (2N, m):
        # row 2i + c holds component c of point i for every column
        xr = torch.view_as_real(qt.reshape(n, m)).permute(0, 2, 1).contiguous()
        yr = torch.empty_like(xr)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.matvec_ptr(xr.data_ptr(), yr.data_ptr(), m, False, near=near, far=far, stream=stream)
        out = torch.view_as_complex(yr.permute(0, 2, 1).contiguous()).reshape(qt.shape)
        return out.cpu().numpy() if is_np else out
