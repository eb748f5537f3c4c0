"""Exact O(N^2) potential sum on the GPU (reference: dense.py:14-33).

``dense_matvec_gpu(points, q)`` computes phi_i = sum_{j != i} -log|x_i - x_j| q_j
in float64 through ``nesa_dense_matvec`` (libnesa_b200.so): the
approximation-error oracle of the NESA product at sizes where the
reference's CPU loop is infeasible (~16 min at 200k,
~27 h at 2M on CPU).  Same contract as the reference: q of shape (N,) (real
or complex; here also (N, k) with k real columns <= 4), ValueError for a
wrong length or coincident points.  There is no CPU fallback.
"""

from __future__ import annotations

import numpy as np

from . import _capi

__all__ = ["dense_matvec_gpu"]


def dense_matvec_gpu(points, q, device: int = 0):
    """phi = K q exactly (float64 on the device); returns numpy, or a CUDA
    tensor when ``q`` is one."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("dense_matvec_gpu needs a CUDA device (no CPU fallback)")
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    n = pts.shape[0]
    if pts.ndim != 2 or pts.shape[1] != 2:
        raise ValueError("points must be (N, 2)")
    is_torch = isinstance(q, torch.Tensor)
    qa = q.detach().cpu().numpy() if is_torch else np.asarray(q)
    if qa.shape[:1] != (n,) or qa.ndim not in (1, 2):
        raise ValueError("q must have one charge per point")
    cplx = np.iscomplexobj(qa)
    cols = qa.reshape(n, -1)
    if cplx:
        cols = np.stack([cols.real, cols.imag], axis=-1).reshape(n, -1)
    cols = np.ascontiguousarray(cols, dtype=np.float64)
    k = cols.shape[1]
    if k > 4:
        raise ValueError("at most 4 real columns per call")
    dev = f"cuda:{device}"
    p_d = torch.from_numpy(pts).to(dev)
    q_d = torch.from_numpy(cols).to(dev)
    phi_d = torch.empty_like(q_d)
    lib = _capi.load()
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream().cuda_stream
        _capi.check(lib.nesa_dense_matvec(p_d.data_ptr(), q_d.data_ptr(), phi_d.data_ptr(), n, k,
                                          stream))
    out = phi_d.cpu().numpy()
    if cplx:
        out = out.reshape(n, -1, 2)
        out = out[..., 0] + 1j * out[..., 1]
    out = out.reshape(qa.shape)
    if is_torch:
        return torch.from_numpy(out).to(q.device)
    return out
