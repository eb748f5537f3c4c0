"""Multi-GPU NESA product: Morton-partitioned leaves, one halo exchange.

The reference has no distributed layer; this follows
SURVEY.md §8e.  Leaves are already in Morton order (quadtree.py:151-183) and
every group covers a contiguous leaf range, so:

* rank r owns a contiguous leaf range, balanced by streamed bytes per leaf
  (near slab n_a * W_a + radiation/reception 2 * n_a * Q);
* its *local groups* are the ancestors of its leaves -- a contiguous id
  range on every level.  The rank computes near / V / U for its leaves and
  C / D / B for its local groups (NesaPlan(leaf_range=...));
* after the upward pass (plan stage 1) a local group's source amplitude s[g]
  is a *partial* sum over the rank's own leaves.  Translation needs the full
  s of every interaction partner, so one exchange completes exactly those:
  each rank packs the partials some other rank needs, one all_gather moves
  them, and each needed group's s is the rank-ordered sum of its
  contributors' partials (deterministic, identical on every rank);
* stage 2 runs translation, downward pass, near field and reception.

Points are owned by exactly one rank, so phi is partitioned; ``gather=True``
sums the per-rank outputs (each point written once) into the full vector.

On GPUs the exchange runs inside the product graph: ``DistNesa`` builds a
distributed plan (C ABI ``nesa_plan_create_dist``) on an NCCL communicator of
its own (``NcclComm``, bootstrapped over the existing torch.distributed
group), and one ``nesa_matvec`` per rank captures pack -> ncclAllGather ->
combine between the upward pass and the translation, with the near field
running concurrently.  The same exchange tables drive a torch-op version
(index_select / all_gather_into_tensor / index adds; ``native=False``) that
runs over gloo in the CPU tests (tests/test_dist_gloo.py) and serves as the
reference for the CUDA pack / combine kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .quadtree import Tree


def leaf_costs(tree: Tree, Q: int) -> np.ndarray:
    """Streamed operator entries per leaf: n_a * W_a + 2 n_a Q."""
    a = tree.arrays
    nl = a.level_count[tree.L]
    n = (a.stop - a.start)[:nl]
    W = np.add.reduceat(n[a.nbr_idx], a.nbr_ptr[:-1]) if a.nbr_idx.size else np.zeros(nl)
    return n * W + 2 * n * Q


def partition_leaves(tree: Tree, world: int, Q: int) -> list[tuple[int, int]]:
    """Contiguous leaf ranges [b, e) per rank, balanced by leaf_costs."""
    nl = tree.arrays.level_count[tree.L]
    if world > nl:
        raise ValueError(f"{world} ranks but only {nl} leaves")
    c = np.cumsum(leaf_costs(tree, Q).astype(np.float64))
    total = c[-1]
    cuts = [0]
    for r in range(1, world):
        k = int(np.searchsorted(c, total * r / world))
        k = max(k, cuts[-1] + 1)
        k = min(k, nl - (world - r))
        cuts.append(k)
    cuts.append(nl)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def local_ranges(tree: Tree, leaf_range: tuple[int, int]) -> dict[int, tuple[int, int]]:
    """Per level: the contiguous id range [lo, hi] of ancestors of the leaves."""
    a = tree.arrays
    lo, hi = leaf_range[0], leaf_range[1] - 1
    out = {}
    for lv in range(tree.L, tree.l0 - 1, -1):
        out[lv] = (lo, hi)
        if lv > tree.l0:
            lo, hi = int(a.parent[lo]), int(a.parent[hi])
    return out


def local_mask(tree: Tree, leaf_range) -> np.ndarray:
    m = np.zeros(tree.arrays.n_groups, bool)
    for lo, hi in local_ranges(tree, leaf_range).values():
        m[lo:hi + 1] = True
    return m


@dataclass
class ExchangePlan:
    """Index tables of the halo exchange for one rank (host arrays)."""

    export_ids: np.ndarray    # (n_export,) groups this rank sends (its partials)
    max_export: int           # buffer rows per rank (padded)
    import_ids: np.ndarray    # (n_import,) groups whose s this rank completes
    contrib: np.ndarray       # (n_import, max_c) rows into [recv rows | local s rows], -1 = none
    n_recv_rows: int          # world * max_export


def build_exchange(tree: Tree, ranges: list[tuple[int, int]], rank: int) -> ExchangePlan:
    """Who sends which partial s to whom."""
    a = tree.arrays
    world = len(ranges)
    G = a.n_groups
    masks = [local_mask(tree, r) for r in ranges]
    # needed(r): interaction partners of r's local groups
    src = np.repeat(np.arange(G), np.diff(a.int_ptr))
    needed = []
    for r in range(world):
        sel = masks[r][src]
        nm = np.zeros(G, bool)
        nm[a.int_idx[sel]] = True
        needed.append(nm)
    n_contrib = np.stack(masks).sum(axis=0)
    # import(r): needed groups whose leaves are not all r's own
    imports = [needed[r] & ~(masks[r] & (n_contrib == 1)) for r in range(world)]
    exports = []
    for r in range(world):
        others = np.zeros(G, bool)
        for r2 in range(world):
            if r2 != r:
                others |= imports[r2]
        exports.append(np.flatnonzero(masks[r] & others))
    max_export = max(1, max(e.size for e in exports))
    pos = [dict(zip(e.tolist(), range(e.size))) for e in exports]
    imp = np.flatnonzero(imports[rank])
    max_c = max(1, int(n_contrib[imp].max()) if imp.size else 1)
    contrib = np.full((imp.size, max_c), -1, np.int64)
    local_base = world * max_export
    for i, g in enumerate(imp.tolist()):
        k = 0
        for r2 in range(world):
            if not masks[r2][g]:
                continue
            if r2 == rank:
                contrib[i, k] = local_base + g          # own partial, read before overwrite
            else:
                contrib[i, k] = r2 * max_export + pos[r2][g]
            k += 1
    return ExchangePlan(export_ids=exports[rank], max_export=max_export, import_ids=imp,
                        contrib=contrib, n_recv_rows=world * max_export)


def _native(s) -> bool:
    return s.is_cuda and s.dtype in (__import__("torch").float32, __import__("torch").float64)


def pack_s(s, xp: ExchangePlan, tensors):
    """This rank's send buffer (max_export, Q*R): its partials others need.
    CUDA: one kernel (nesa_exchange_pack); CPU (gloo tests): torch ops."""
    import torch
    exp_ids = tensors[0]
    if _native(s):
        from . import _capi
        send = torch.empty((xp.max_export, s.shape[1]), dtype=s.dtype, device=s.device)
        _capi.check(_capi.load().nesa_exchange_pack(
            s.data_ptr(), exp_ids.data_ptr() if exp_ids.numel() else None, exp_ids.numel(),
            xp.max_export, s.shape[1], int(s.dtype == torch.float64), send.data_ptr(),
            torch.cuda.current_stream(s.device).cuda_stream))
        return send
    send = torch.zeros((xp.max_export, s.shape[1]), dtype=s.dtype, device=s.device)
    if exp_ids.numel():
        send[:exp_ids.numel()] = s.index_select(0, exp_ids)
    return send


def combine_s(s, xp: ExchangePlan, recv, tensors) -> None:
    """s[g] = rank-ordered sum of the contributors' partials, for imported g."""
    import torch
    _, imp_ids, contrib = tensors
    if imp_ids.numel() == 0:
        return
    if _native(s):
        from . import _capi
        _capi.check(_capi.load().nesa_exchange_combine(
            s.data_ptr(), recv.data_ptr(), imp_ids.data_ptr(), contrib.data_ptr(), imp_ids.numel(),
            contrib.shape[1], recv.shape[0], s.shape[1], int(s.dtype == torch.float64),
            torch.cuda.current_stream(s.device).cuda_stream))
        return
    pool = torch.cat((recv, s), 0)                      # rows: recv | local s (all G)
    acc = torch.zeros((imp_ids.numel(), s.shape[1]), dtype=s.dtype, device=s.device)
    zero = torch.zeros((), dtype=s.dtype, device=s.device)
    for k in range(contrib.shape[1]):                   # fixed rank order
        col = contrib[:, k]
        rows = pool.index_select(0, col.clamp(min=0))
        acc += torch.where((col >= 0)[:, None], rows, zero)
    s.index_copy_(0, imp_ids, acc)


def exchange_s(s, xp: ExchangePlan, group=None, tensors=None):
    """Complete the needed source amplitudes in place (one all_gather).

    ``s`` is a torch tensor viewed as (G, Q*R) (device or CPU).  ``tensors``
    caches the device copies of the index tables.
    """
    import torch
    import torch.distributed as dist
    if tensors is None:
        tensors = exchange_tensors(xp, s.device)
    send = pack_s(s, xp, tensors)
    world = dist.get_world_size(group)
    recv = torch.empty((world * xp.max_export, s.shape[1]), dtype=s.dtype, device=s.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    combine_s(s, xp, recv, tensors)


def exchange_tensors(xp: ExchangePlan, device):
    import torch
    return (torch.as_tensor(xp.export_ids, dtype=torch.long, device=device),
            torch.as_tensor(xp.import_ids, dtype=torch.long, device=device),
            torch.as_tensor(xp.contrib, dtype=torch.long, device=device))


class NcclComm:
    """An NCCL communicator of the product library (nesa_nccl_comm_init),
    bootstrapped over an initialised torch.distributed group: rank 0 draws
    the unique id, the group broadcasts it."""

    def __init__(self, device: int, group=None):
        import ctypes

        import torch.distributed as dist
        from . import _capi
        self.lib = _capi.load()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = bytearray(128)
        if rank == 0:
            buf = (ctypes.c_char * 128)()
            _capi.check(self.lib.nesa_nccl_unique_id(buf, 128))
            uid = bytearray(buf.raw)
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        raw = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        _capi.check(self.lib.nesa_nccl_comm_init(raw, world, rank, device, ctypes.byref(h)))
        self.handle = h.value
        self.rank, self.world = rank, world

    def close(self) -> None:
        if self.handle:
            self.lib.nesa_nccl_comm_destroy(self.handle)
            self.handle = None


class DistNesa:
    """One rank of a multi-GPU product (torch.distributed already initialised).

    ``native`` (default on CUDA): the distributed plan with the exchange in
    its graph -- one ``nesa_matvec`` launch per product and rank.  Otherwise
    the stage-1 / Python exchange / stage-2 sequence (the CPU-testable path).
    """

    def __init__(self, tree: Tree, ops, dtype: str = "f32", device: int = 0, group=None,
                 native: bool = True):
        import torch.distributed as dist
        from .plan import NesaPlan
        self.tree = tree
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        params = getattr(ops, "params", ops)
        self.Q = params.Q
        self.ranges = partition_leaves(tree, self.world, self.Q)
        self.leaf_range = self.ranges[self.rank]
        self.xp = build_exchange(tree, self.ranges, self.rank)
        self.comm = NcclComm(device, group) if native else None
        self.plan = NesaPlan(tree, ops, dtype=dtype, device=device, leaf_range=self.leaf_range,
                             comm=self.comm.handle if native else None, rank=self.rank,
                             nranks=self.world, exchange=self.xp if native else None)
        self.native = native
        self._tensors = None
        self.device = device

    def close(self) -> None:
        self.plan.close()
        if self.comm is not None:
            self.comm.close()

    def matvec_ptr(self, q_ptr: int, phi_ptr: int, nrhs: int, is_complex: bool,
                   near: bool = True, far: bool = True, stream: int = 0, profile=False) -> None:
        import torch
        R = nrhs * (2 if is_complex else 1)
        if self.native:
            # one graph: gather, near || radiation + upward pass, exchange over
            # NCCL, translation + downward pass, reception (this rank's points)
            self.plan.matvec_ptr(q_ptr, phi_ptr, nrhs, is_complex, near=near, far=far, stream=stream,
                                 profile=profile)
            return
        self.plan.matvec_ptr(q_ptr, phi_ptr, nrhs, is_complex, near=near, far=far,
                             stream=stream, stage=1)
        if far:
            s_ptr = self.plan.s_dev_ptr(R)
            G = self.tree.arrays.n_groups
            dt = torch.float64 if self.plan.dtype == "f64" else torch.float32
            s = _tensor_from_ptr(s_ptr, (G, self.Q * R), dt, self.device)
            ext = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
            with torch.cuda.stream(ext):
                if self._tensors is None:
                    self._tensors = exchange_tensors(self.xp, s.device)
                exchange_s(s, self.xp, self.group, self._tensors)
        self.plan.matvec_ptr(q_ptr, phi_ptr, nrhs, is_complex, near=near, far=far,
                             stream=stream, stage=2)

    def matvec(self, q, gather: bool = True):
        """q: CUDA tensor (N,) / (N, nrhs) on this rank's device."""
        import torch
        import torch.distributed as dist
        phi = torch.zeros_like(q)
        nrhs = 1 if q.dim() == 1 else q.shape[1]
        self.matvec_ptr(q.data_ptr(), phi.data_ptr(), nrhs, q.is_complex(),
                        stream=torch.cuda.current_stream().cuda_stream)
        if gather:
            view = torch.view_as_real(phi) if phi.is_complex() else phi
            dist.all_reduce(view, group=self.group)
        return phi


def _tensor_from_ptr(ptr: int, shape, dtype, device: int):
    """Non-owning torch view of plan-owned device memory."""
    import torch
    n = int(np.prod(shape))
    itemsize = torch.tensor([], dtype=dtype).element_size()

    class _Holder:
        __cuda_array_interface__ = {
            "shape": (n,), "typestr": "<f8" if itemsize == 8 else "<f4",
            "data": (ptr, False), "version": 3, "strides": None,
        }

    return torch.as_tensor(_Holder(), device=f"cuda:{device}").view(*shape)
