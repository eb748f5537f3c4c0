"""The NESA matrix-vector product on the GPU -- drop-in for taskfmm.fastmvp.

Same call shapes as the reference (/root/reference/pkg/src/taskfmm/
fastmvp.py:124-187):

* ``mvp(tree, ops, q, runtime=None, vec=None, near=True, far=True)``
* ``mvp_serial(tree, ops, q, near=True, far=True)``  (same product; the GPU
  has no serial/parallel distinction, the name is kept for drop-in use)
* ``task_counts(tree)``

``q`` may be a numpy array (returns numpy, like the reference) or a CUDA
torch tensor (returns a CUDA tensor, no host copies).  Real or complex,
shape (N,) or (N, nrhs).  float64 / complex128 run the float64 plan,
float32 / complex64 the float32 plan.  A wrong length raises ``ValueError``
as fastmvp.py:128-129 does.  Work vectors are plan-owned and rewritten on
every call (StageVectors.reset semantics, fastmvp.py:42-45), so repeated
calls never see stale sums.

There is no CPU fallback: without the CUDA library or a GPU these raise.
"""

from __future__ import annotations

import numpy as np

from .operators import NesaParams, OperatorSet, OperatorTables
from .plan import NesaPlan
from .quadtree import Tree, TreeArrays

__all__ = ["mvp", "mvp_serial", "task_counts", "get_plan", "get_lanes", "as_tree", "RhsLanes"]


def as_tree(tree) -> Tree:
    """Accept our Tree or a reference taskfmm Tree (groups list) unchanged."""
    if isinstance(tree, Tree):
        return tree
    cached = getattr(tree, "_nesa_tree", None)
    if cached is not None:
        return cached
    groups = tree.groups
    G = len(groups)
    lvl = np.array([g.level for g in groups], np.int32)
    ix = np.array([g.ix for g in groups], np.int64)
    iy = np.array([g.iy for g in groups], np.int64)
    start = np.array([g.start for g in groups], np.int64)
    stop = np.array([g.stop for g in groups], np.int64)
    parent = np.array([-1 if g.parent is None else g.parent for g in groups], np.int64)
    cf = np.array([g.children[0] if g.children else -1 for g in groups], np.int64)
    nc = np.array([len(g.children) for g in groups], np.int64)
    box = np.array([[g.box.xmin, g.box.ymin, g.box.xmax, g.box.ymax] for g in groups])
    leaves = tree.level_ids[tree.L]
    nbr_ptr = np.cumsum([0] + [len(groups[i].neighbors) for i in leaves]).astype(np.int64)
    nbr_idx = np.array([b for i in leaves for b in groups[i].neighbors], np.int64)
    int_ptr = np.cumsum([0] + [len(g.interaction) for g in groups]).astype(np.int64)
    int_idx = np.array([b for g in groups for b in g.interaction], np.int64)
    lf = {lv: min(ids) for lv, ids in tree.level_ids.items()}
    lc = {lv: len(ids) for lv, ids in tree.level_ids.items()}
    arrays = TreeArrays(level=lvl, ix=ix, iy=iy, start=start, stop=stop, parent=parent,
                        child_first=cf, n_children=nc, box=box, level_first=lf,
                        level_count=lc, nbr_ptr=nbr_ptr, nbr_idx=nbr_idx,
                        int_ptr=int_ptr, int_idx=int_idx)
    out = Tree(params=tree.params, l0=tree.l0, L=tree.L, root_origin=tree.root_origin,
               root_side=tree.root_side, arrays=arrays, perm=np.asarray(tree.perm),
               points=np.asarray(tree.points))
    try:
        tree._nesa_tree = out
    except AttributeError:
        pass
    return out


def get_plan(tree, ops, dtype: str = "f64", device: int = 0, wide: bool = False) -> NesaPlan:
    """Cached plan for (tree, ops, dtype, device); built on first use.

    ``wide``: the plan for products of more than 4 real columns -- stored
    V / U blocks, so the far field runs as batched GEMMs over 128-column
    passes (for a host OperatorSet that is the ordinary plan)."""
    t = as_tree(tree)
    cache = getattr(t, "_nesa_plans", None)
    if cache is None:
        cache = {}
        t._nesa_plans = cache
    if wide and isinstance(ops, OperatorSet):
        wide = False
    key = (id(ops), dtype, device, wide)
    ent = cache.get(key)
    if ent is None or ent[0] is not ops:
        if not isinstance(ops, (OperatorSet, OperatorTables, NesaParams)):
            ops_in = _adopt_opset(ops)
        else:
            ops_in = ops
        ent = (ops, NesaPlan(t, ops_in, dtype=dtype, device=device, stored_vu=wide))
        cache[key] = ent
    return ent[1]


class RhsLanes:
    """Many right-hand sides spread over ``lanes`` plans of the same problem
    (each with its own workspace and CUDA graphs) on ``lanes`` streams.

    The far field runs in blocks of <= 4 real columns, and every block walks
    the latency-bound far-field chain again; blocks of different lanes run
    concurrently, so their chains overlap.  On float32 plans with tensor
    cores the near field is ONE tcgen05 GEMM over all columns
    (nesa_matvec_near_wide, operator streamed once) after the lanes join, and
    the extra lanes are far-only plans (no near operator uploaded).  Otherwise
    each block also carries its near field.  The column ranges are multiples
    of 4, so the block decomposition -- and every result bit -- is that of
    the single-plan product.
    """

    def __init__(self, plan: NesaPlan, lanes: int):
        import torch
        self.wide = plan.stat("near_wide") == 1
        self.plans = [plan] + [NesaPlan(plan.tree, plan.ops_in, dtype=plan.dtype,
                                        device=plan.device, far_only=self.wide)
                               for _ in range(lanes - 1)]
        self.streams = [torch.cuda.Stream(plan.device) for _ in range(lanes)]
        self.events = [torch.cuda.Event() for _ in range(lanes)]

    def matvec_ptr(self, q_ptr: int, phi_ptr: int, nrhs: int, is_complex: bool,
                   near: bool = True, far: bool = True, stream: int = 0) -> None:
        import torch
        rt = nrhs * (2 if is_complex else 1)
        blocks = -(-rt // 4)
        lanes = min(len(self.plans), blocks)
        per = -(-blocks // lanes) * 4
        caller = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        wide_near = near and self.wide
        fork = torch.cuda.Event()
        fork.record(caller)
        used = []
        for k in range(lanes):
            c0 = k * per
            n = min(per, rt - c0)
            if n <= 0:
                break
            s = self.streams[k]
            s.wait_event(fork)
            self.plans[k].matvec_cols_ptr(q_ptr, phi_ptr, rt, c0, n, near=near and not wide_near,
                                          far=far, stream=s.cuda_stream)
            self.events[k].record(s)
            used.append(k)
        for k in used:
            caller.wait_event(self.events[k])
        if wide_near:
            self.plans[0].near_wide_ptr(q_ptr, phi_ptr, rt, 0, rt, stream=caller.cuda_stream)


def get_lanes(tree, ops, dtype: str = "f64", device: int = 0, lanes: int | None = None) -> RhsLanes:
    """Cached RhsLanes for (tree, ops, dtype, device); lane 0 is get_plan's."""
    import os
    if lanes is None:
        # C5 (200k points, 64 plane waves): 1 / 2 / 4 / 8 / 16 lanes ->
        # 10.5 / 8.9 / 6.0 / 5.1 / 5.0 ms (tools/lanes_sweep.py)
        lanes = max(1, int(os.environ.get("NESA_RHS_LANES", "8")))
    plan = get_plan(tree, ops, dtype=dtype, device=device)
    ent = getattr(plan, "_lanes", None)
    if ent is None or len(ent.plans) != lanes:
        ent = RhsLanes(plan, lanes)
        plan._lanes = ent
    return ent


def _adopt_opset(ops) -> OperatorSet:
    """A reference taskfmm OperatorSet -> ours (same dicts, shared matrices)."""
    p = ops.params
    params = NesaParams(Q=p.Q, oversampling=p.oversampling, rho_out_aux=p.rho_out_aux,
                        rho_out_check=p.rho_out_check, rho_in_check=p.rho_in_check,
                        rho_in_aux=p.rho_in_aux, pinv_cutoff=p.pinv_cutoff)
    return OperatorSet(params=params, V=ops.V, U=ops.U, C=ops.C, B=ops.B, D=ops.D,
                       near=ops.near)


def _torch():
    import torch
    return torch


def mvp(tree, ops, q, runtime=None, vec=None, near: bool = True, far: bool = True,
        device: int | None = None):
    """phi = K~ q in the original point order (fastmvp.py:124-139 contract).

    ``runtime`` and ``vec`` are accepted for signature compatibility: the
    task runtime is replaced by the plan's CUDA graph, the stage vectors by
    plan-owned device workspace.
    """
    torch = _torch()
    t = as_tree(tree)
    is_torch = isinstance(q, torch.Tensor)
    shape = tuple(q.shape)
    if len(shape) not in (1, 2) or shape[0] != t.n_points:
        raise ValueError("q must have one charge per point")
    nrhs = 1 if len(shape) == 1 else shape[1]
    if is_torch:
        is_complex = q.is_complex()
        single = q.dtype in (torch.float32, torch.complex64)
        dev = q.device.index if q.is_cuda else (device or 0)
    else:
        q = np.asarray(q)
        is_complex = np.iscomplexobj(q)
        single = q.dtype in (np.float32, np.complex64)
        dev = device or 0
    dtype = "f32" if single else "f64"
    if not torch.cuda.is_available():
        raise RuntimeError("mvp needs a CUDA device (no CPU fallback)")
    plan = get_plan(t, ops, dtype=dtype, device=dev)
    tdt = {("f64", False): torch.float64, ("f64", True): torch.complex128,
           ("f32", False): torch.float32, ("f32", True): torch.complex64}[(dtype, is_complex)]
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        on_host = (not is_torch) or not q.is_cuda
        if is_torch:
            qd = q.to(device=f"cuda:{dev}", dtype=tdt, non_blocking=True).contiguous()
        else:
            qd = torch.from_numpy(np.ascontiguousarray(q)).to(f"cuda:{dev}", dtype=tdt)
        phi = torch.empty_like(qd)
        wide = nrhs * (2 if is_complex else 1) > 4
        if wide and far:
            # many right-hand sides: the far field as batched GEMMs over all
            # columns, the near field as one tensor-core GEMM (float32)
            wplan = get_plan(t, ops, dtype=dtype, device=dev, wide=True)
        if wide and far and wplan.stat("far_wide") == 1 and (not near or dtype == "f32"):
            wplan.matvec_ptr(qd.data_ptr(), phi.data_ptr(), nrhs, is_complex, near=near, far=far,
                             stream=stream.cuda_stream)
        elif wide:   # several blocks of <= 4 columns, spread over lanes
            get_lanes(t, ops, dtype=dtype, device=dev).matvec_ptr(
                qd.data_ptr(), phi.data_ptr(), nrhs, is_complex, near=near, far=far,
                stream=stream.cuda_stream)
        else:
            plan.matvec_ptr(qd.data_ptr(), phi.data_ptr(), nrhs, is_complex, near=near, far=far,
                            stream=stream.cuda_stream)
        if not on_host:
            return phi
        if is_torch:        # CPU tensor in -> CPU tensor out (pinned if the input was)
            out = torch.empty(phi.shape, dtype=phi.dtype, pin_memory=q.is_pinned())
            out.copy_(phi, non_blocking=True)
            stream.synchronize()
            return out
        return phi.cpu().numpy()


def mvp_serial(tree, ops, q, near: bool = True, far: bool = True):
    """Same product as :func:`mvp` (fastmvp.py:142-172 signature)."""
    return mvp(tree, ops, q, near=near, far=far)


def task_counts(tree) -> dict:
    """Per-stage gemv counts of the reference's task graph (fastmvp.py:175-187).

    On the GPU each of these becomes a row of a batched launch; the counts
    are the work the plan performs per product.
    """
    t = as_tree(tree)
    a = t.arrays
    n_leaves = a.level_count[t.L]
    n_edges = sum(a.level_count[lv] for lv in range(t.l0 + 1, t.L + 1))
    return {
        "near": int(a.nbr_ptr[-1]),
        "radiation": int(n_leaves),
        "source-transfer": int(n_edges),
        "translation": int(a.int_ptr[-1]),
        "potential-transfer": int(n_edges),
        "reception": int(n_leaves),
    }
