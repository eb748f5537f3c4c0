"""Pipelined products from host memory: H2D / product / D2H of successive
calls overlap.

``fastmvp.mvp`` is synchronous: each call copies q in, runs the product and
copies phi out before returning, so the PCIe transfers (16 MB each way at
N = 2M complex64) serialise with the product.  A caller with a stream of
independent right-hand sides -- several systems solved side by side, a
serving loop -- uses this class instead:

    pipe = MvpPipeline(tree, ops, dtype="f32", is_complex=True)
    for q_host, phi_host in pairs:          # pinned CPU tensors
        pipe.submit(q_host, phi_host)       # returns at once
    pipe.synchronize()                      # every phi_host is written

Streams: one for H2D copies, one per compute slot, one for D2H copies.
Submission k uses slot k % slots.  A slot is a complete plan (its own
workspace and CUDA graph; the operator data is uploaded per slot), so with
slots >= 2 the products of consecutive submissions may also overlap each
other.  One slot is the default: a C4 product already keeps the whole GPU
busy (near field beside the far-field chain), and two concurrent products
only contend (measured 1845 vs 1697 products/s end to end with 1 vs 2
slots); the transfers still overlap the neighbouring products.  Events order reuse of every
buffer (an upload never overwrites an input a product still reads, a
product never overwrites a result still being downloaded).  Each result is
bitwise identical to ``mvp`` for the same plan parameters.
"""

from __future__ import annotations

from .fastmvp import as_tree, get_plan
from .plan import NesaPlan

__all__ = ["MvpPipeline"]


class MvpPipeline:
    """Overlapped host-to-host products for one (tree, ops) pair."""

    def __init__(self, tree, ops, dtype: str = "f32", is_complex: bool = True, nrhs: int = 1,
                 device: int = 0, slots: int = 1):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("MvpPipeline needs a CUDA device (no CPU fallback)")
        if slots < 1:
            raise ValueError("slots must be >= 1")
        self.tree = as_tree(tree)
        # slot 0 shares the cached plan of mvp(); further slots are private
        self.plans = [get_plan(self.tree, ops, dtype=dtype, device=device)]
        for _ in range(slots - 1):
            self.plans.append(NesaPlan(self.tree, self.plans[0].ops_in, dtype=dtype,
                                       device=device))
        self.device = device
        self.slots = slots
        self.nrhs = nrhs
        self.is_complex = is_complex
        n = self.tree.n_points
        tdt = {("f64", False): torch.float64, ("f64", True): torch.complex128,
               ("f32", False): torch.float32, ("f32", True): torch.complex64}[(dtype, is_complex)]
        self.dtype = tdt
        shape = (n,) if nrhs == 1 else (n, nrhs)
        self.shape = shape
        dev = f"cuda:{device}"
        # two input / output buffers per slot: the upload of k + slots overlaps product k
        nb = 2 * slots
        self.q_dev = [torch.empty(shape, dtype=tdt, device=dev) for _ in range(nb)]
        self.phi_dev = [torch.empty(shape, dtype=tdt, device=dev) for _ in range(nb)]
        self.s_h2d = torch.cuda.Stream(device)
        self.s_comp = [torch.cuda.Stream(device) for _ in range(slots)]
        self.s_d2h = torch.cuda.Stream(device)
        self.ev_in = [torch.cuda.Event() for _ in range(nb)]     # upload done
        self.ev_used = [torch.cuda.Event() for _ in range(nb)]   # product done
        self.ev_out = [torch.cuda.Event() for _ in range(nb)]    # download done
        self.k = 0

    def submit(self, q_host, phi_host) -> None:
        """Queue one product: q_host -> phi_host (pinned CPU tensors of the
        pipeline's shape and dtype).  Returns without waiting."""
        import torch
        if tuple(q_host.shape) != self.shape or tuple(phi_host.shape) != self.shape:
            raise ValueError("q must have one charge per point")
        if q_host.dtype != self.dtype or phi_host.dtype != self.dtype:
            raise ValueError(f"expected {self.dtype}")
        nb = len(self.q_dev)
        b = self.k % nb
        slot = self.k % self.slots
        reuse = self.k >= nb
        qd, pd = self.q_dev[b], self.phi_dev[b]
        comp = self.s_comp[slot]
        # upload into buffer b once the product that last read it is done
        if reuse:
            self.s_h2d.wait_event(self.ev_used[b])
        with torch.cuda.stream(self.s_h2d):
            qd.copy_(q_host, non_blocking=True)
            self.ev_in[b].record(self.s_h2d)
        # product after its upload and after the download that last read phi b
        comp.wait_event(self.ev_in[b])
        if reuse:
            comp.wait_event(self.ev_out[b])
        self.plans[slot].matvec_ptr(qd.data_ptr(), pd.data_ptr(), self.nrhs, self.is_complex,
                                    stream=comp.cuda_stream)
        self.ev_used[b].record(comp)
        # download once the product is done
        self.s_d2h.wait_event(self.ev_used[b])
        with torch.cuda.stream(self.s_d2h):
            phi_host.copy_(pd, non_blocking=True)
            self.ev_out[b].record(self.s_d2h)
        self.k += 1

    def synchronize(self) -> None:
        """Wait until every submitted product's result is in host memory."""
        self.s_d2h.synchronize()
