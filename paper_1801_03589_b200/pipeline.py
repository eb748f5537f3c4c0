"""Pipelined products from host memory: H2D / product / D2H of successive
calls overlap.

``fastmvp.mvp`` is synchronous: each call copies q in, runs the product and
copies phi out before returning, so the PCIe transfers (16 MB each way at
N = 2M complex64) serialise with the product.  A caller with a stream of
right-hand sides -- an iterative solver on several systems, a serving loop --
uses this class instead:

    pipe = MvpPipeline(tree, ops, dtype="f32", is_complex=True)
    for q_host, phi_host in pairs:          # pinned CPU tensors
        pipe.submit(q_host, phi_host)       # returns at once
    pipe.synchronize()                      # every phi_host is written

Three CUDA streams: H2D copies (``depth`` device input slots), the product
(the plan's CUDA graph, strictly in submission order: the plan's workspace
is shared), and D2H copies.  While product k runs, the input of k+1 is
uploaded and the result of k-1 downloaded.  Events order slot reuse, so a
slot is never overwritten while a product or a download still reads it.
Results are identical to ``mvp`` (same plan, same graph).
"""

from __future__ import annotations

from .fastmvp import as_tree, get_plan

__all__ = ["MvpPipeline"]


class MvpPipeline:
    """Overlapped host-to-host products for one (tree, ops) pair."""

    def __init__(self, tree, ops, dtype: str = "f32", is_complex: bool = True, nrhs: int = 1,
                 device: int = 0, depth: int = 2):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("MvpPipeline needs a CUDA device (no CPU fallback)")
        if depth < 2:
            raise ValueError("depth must be >= 2")
        self.tree = as_tree(tree)
        self.plan = get_plan(self.tree, ops, dtype=dtype, device=device)
        self.device = device
        self.depth = depth
        self.nrhs = nrhs
        self.is_complex = is_complex
        n = self.tree.n_points
        tdt = {("f64", False): torch.float64, ("f64", True): torch.complex128,
               ("f32", False): torch.float32, ("f32", True): torch.complex64}[(dtype, is_complex)]
        self.dtype = tdt
        shape = (n,) if nrhs == 1 else (n, nrhs)
        self.shape = shape
        dev = f"cuda:{device}"
        self.q_dev = [torch.empty(shape, dtype=tdt, device=dev) for _ in range(depth)]
        self.phi_dev = [torch.empty(shape, dtype=tdt, device=dev) for _ in range(depth)]
        self.s_h2d = torch.cuda.Stream(device)
        self.s_comp = torch.cuda.Stream(device)
        self.s_d2h = torch.cuda.Stream(device)
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]     # upload k done
        self.ev_used = [torch.cuda.Event() for _ in range(depth)]   # product k done
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]    # download k done
        self.k = 0

    def submit(self, q_host, phi_host) -> None:
        """Queue one product: q_host -> phi_host (pinned CPU tensors of the
        pipeline's shape and dtype).  Returns without waiting."""
        import torch
        if tuple(q_host.shape) != self.shape or tuple(phi_host.shape) != self.shape:
            raise ValueError("q must have one charge per point")
        if q_host.dtype != self.dtype or phi_host.dtype != self.dtype:
            raise ValueError(f"expected {self.dtype}")
        slot = self.k % self.depth
        first = self.k < self.depth
        qd, pd = self.q_dev[slot], self.phi_dev[slot]
        # upload into the slot once product k - depth has consumed it
        if not first:
            self.s_h2d.wait_event(self.ev_used[slot])
        with torch.cuda.stream(self.s_h2d):
            qd.copy_(q_host, non_blocking=True)
            self.ev_in[slot].record(self.s_h2d)
        # product k after its upload and after download k - depth left the slot
        self.s_comp.wait_event(self.ev_in[slot])
        if not first:
            self.s_comp.wait_event(self.ev_out[slot])
        self.plan.matvec_ptr(qd.data_ptr(), pd.data_ptr(), self.nrhs, self.is_complex,
                             stream=self.s_comp.cuda_stream)
        self.ev_used[slot].record(self.s_comp)
        # download once the product is done
        self.s_d2h.wait_event(self.ev_used[slot])
        with torch.cuda.stream(self.s_d2h):
            phi_host.copy_(pd, non_blocking=True)
            self.ev_out[slot].record(self.s_d2h)
        self.k += 1

    def synchronize(self) -> None:
        """Wait until every submitted product's result is in host memory."""
        self.s_d2h.synchronize()
