"""Iterative solver around the GPU NESA product.

The reference only multiplies (no solver); the paper names the
product as the inner kernel of an iterative solver.  This
is restarted GMRES for

    (shift * I + K~) x = b

with every product on the GPU (``NesaPlan.matvec_ptr`` on device tensors, no
host copies of the N-vectors) and several right-hand sides solved side by
side: the columns run independent Arnoldi processes in lockstep, so each
iteration is ONE multi-column product (the plan streams the near-field
operator once for up to 4 real columns, see nesa_plan.cu run_matvec).

Orthogonalisation is classical Gram-Schmidt applied twice (CGS2).  For one
complex column it is the library's fused step (``nesa_gs_step``: three
passes over the basis, the Hessenberg column written on the device, no
host round trip); the host applies the Givens rotations of iteration k while
the GPU already runs iteration k+1 (the convergence test lags one iteration,
the extra product is discarded).  Several columns run in lockstep with
batched torch projections.  ``shift`` turns the first-kind log-kernel system
into a second-kind one when wanted (the first-kind system is ill conditioned
and converges slowly, as for any first-kind integral equation).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .fastmvp import as_tree, get_plan

__all__ = ["gmres", "GmresResult"]


@dataclass
class GmresResult:
    x: object                 # solution, same kind (numpy / torch) and shape as b
    iterations: int           # inner iterations (products) performed
    residuals: np.ndarray     # final relative residual per column (true, recomputed)
    converged: np.ndarray     # per column
    history: list             # estimated relative residual per iteration, (n_iter, m)


def _givens(a: complex, b: complex):
    """(c, s) with [c, s; -conj(s), c] [a; b] = [r; 0]."""
    if b == 0:
        return 1.0, 0.0
    if a == 0:
        return 0.0, 1.0
    r = np.hypot(abs(a), abs(b))
    c = abs(a) / r
    s = (a / abs(a)) * np.conj(b) / r
    return c, s


def _arnoldi_fused(A, V, H, cs, sn, g, k_max, bnorm, done, tol, history, iters, maxiter, w_buf,
                   gs_work, lib, stream, is_f64, shift=0.0):
    """One restart cycle for one complex column: products and CGS2 steps on
    the device (nesa_gs_step), Givens rotations on the host one iteration
    behind.  Returns the number of basis columns to use."""
    import torch
    from . import _capi
    n = V.shape[1]
    stride = V[1].data_ptr() - V[0].data_ptr()
    stride //= V.element_size() // 2           # in real elements
    hdev = torch.zeros((k_max, 2 * (k_max + 1)), dtype=torch.float64, device=V.device)
    hhost = torch.zeros((k_max, 2 * (k_max + 1)), dtype=torch.float64).pin_memory()
    evs = [torch.cuda.Event() for _ in range(k_max)]

    def launch(k):
        A(V[k], w_buf, with_shift=False)  # the shift is added inside the first GS pass
        rc = lib.nesa_gs_step_shifted(V.data_ptr(), stride, k + 1, w_buf.data_ptr(), V[k + 1].data_ptr(),
                                      n, int(is_f64), float(shift), gs_work.data_ptr(), hdev[k].data_ptr(),
                                      stream.cuda_stream)
        if rc:
            raise RuntimeError(lib.nesa_gs_last_error().decode())
        hhost[k].copy_(hdev[k], non_blocking=True)
        evs[k].record(stream)

    budget = maxiter - iters
    k_run = min(k_max, budget)
    if k_run <= 0:
        return 0, 0
    launch(0)
    launched = 1
    k_used = 0
    for k in range(k_run):
        if k + 1 < k_run:
            launch(k + 1)       # the next product runs while the host rotates column k
            launched += 1
        evs[k].synchronize()
        hv = hhost[k].numpy()
        col = hv[0:2 * (k + 2):2] + 1j * hv[1:2 * (k + 2):2]
        H[:k + 2, k, 0] = col
        for j in range(k):
            a0, a1 = H[j, k, 0], H[j + 1, k, 0]
            H[j, k, 0] = cs[j, 0] * a0 + sn[j, 0] * a1
            H[j + 1, k, 0] = -np.conj(sn[j, 0]) * a0 + cs[j, 0] * a1
        cc, ss = _givens(H[k, k, 0], H[k + 1, k, 0])
        cs[k, 0], sn[k, 0] = cc, ss
        H[k, k, 0] = cc * H[k, k, 0] + ss * H[k + 1, k, 0]
        H[k + 1, k, 0] = 0
        g[k + 1, 0] = -np.conj(ss) * g[k, 0]
        g[k, 0] = cc * g[k, 0]
        k_used = k + 1
        est = np.abs(g[k + 1]) / bnorm
        est[done] = 0.0
        history.append(est.copy())
        if (est <= tol).all():
            break
    stream.synchronize()
    return k_used, launched


def gmres(tree, ops, b, shift: float = 0.0, tol: float = 1e-6, restart: int = 40,
          maxiter: int = 400, x0=None, device: int | None = None,
          orthogonalise: str = "auto") -> GmresResult:
    """Restarted GMRES on the GPU for (shift I + K~) x = b.

    b: (N,) or (N, m), numpy or torch (CPU or CUDA); real or complex; float32
    / complex64 use the float32 plan, float64 / complex128 the float64 plan.
    Columns stop updating once their relative residual is below ``tol``.
    """
    import torch
    t = as_tree(tree)
    is_torch = isinstance(b, torch.Tensor)
    on_host = (not is_torch) or not b.is_cuda
    if is_torch:
        dev = b.device.index if b.is_cuda else (device or 0)
        bd = b.to(f"cuda:{dev}")
    else:
        dev = device or 0
        bd = torch.from_numpy(np.ascontiguousarray(b)).to(f"cuda:{dev}")
    if bd.shape[0] != t.n_points or bd.dim() not in (1, 2):
        raise ValueError("b must have one value per point")
    vec = bd.dim() == 1
    B = bd.reshape(t.n_points, -1).contiguous()
    m = B.shape[1]
    single = B.dtype in (torch.float32, torch.complex64)
    is_complex = B.is_complex()
    plan = get_plan(t, ops, dtype="f32" if single else "f64", device=dev)
    stream = torch.cuda.current_stream(dev)

    def A(X, Y=None, with_shift=True):
        Y = torch.empty_like(X) if Y is None else Y
        plan.matvec_ptr(X.data_ptr(), Y.data_ptr(), m, is_complex, stream=stream.cuda_stream)
        if shift and with_shift:
            Y.add_(X, alpha=shift)
        return Y

    # "auto": the fused device step for one complex column, batched torch
    # projections otherwise ("torch" forces the latter)
    fused = orthogonalise != "torch" and m == 1 and is_complex and restart < 128
    if fused:
        from . import _capi
        lib = _capi.load()
        gs_work = torch.zeros(int(lib.nesa_gs_work_bytes()), dtype=torch.uint8, device=B.device)
        w_buf = torch.empty_like(B)

    def cnorm(X):                      # per-column 2-norms, float64 on host
        return torch.linalg.vector_norm(X, dim=0).double().cpu().numpy()

    X = torch.zeros_like(B) if x0 is None else (
        x0 if isinstance(x0, torch.Tensor) else torch.from_numpy(np.asarray(x0))
    ).to(B.device, B.dtype).reshape(B.shape).clone()
    bnorm = cnorm(B)
    bnorm[bnorm == 0] = 1.0
    hdt = np.complex128 if is_complex else np.float64
    history = []
    iters = 0
    done = np.zeros(m, bool)
    while iters < maxiter and not done.all():
        Rv = B - A(X) if iters or x0 is not None else B.clone()
        if iters or x0 is not None:
            iters += 1
        beta = cnorm(Rv)
        done |= beta / bnorm <= tol
        if done.all():
            break
        k_max = min(restart, maxiter - iters)
        if k_max <= 0:
            break
        V = torch.empty((k_max + 1,) + tuple(B.shape), dtype=B.dtype, device=B.device)
        scale = torch.as_tensor(np.where(beta > 0, 1.0 / np.maximum(beta, 1e-300), 0.0),
                                device=B.device, dtype=B.real.dtype if is_complex else B.dtype)
        V[0] = Rv * scale
        H = np.zeros((k_max + 1, k_max, m), hdt)
        cs = np.zeros((k_max, m))
        sn = np.zeros((k_max, m), hdt)
        g = np.zeros((k_max + 1, m), hdt)
        g[0] = beta
        k_used = 0
        if fused:
            k_used, launched = _arnoldi_fused(A, V, H, cs, sn, g, k_max, bnorm, done, tol, history,
                                              iters, maxiter, w_buf, gs_work, lib, stream,
                                              is_f64=not single, shift=shift)
            iters += launched
        for k in range(0 if not fused else k_max, k_max):
            W = A(V[k])
            iters += 1
            # classical Gram-Schmidt, twice (CGS2): two batched projections
            # against the whole basis per iteration, one host transfer
            Vk = V[:k + 1]
            if m == 1:   # GEMV (cuBLAS) on the (k+1, N) basis
                V2, w = Vk.reshape(k + 1, -1), W.reshape(-1)
                Vc = V2.conj() if is_complex else V2
                h1 = torch.mv(Vc, w)
                w -= torch.mv(V2.t(), h1)
                h2 = torch.mv(Vc, w)
                w -= torch.mv(V2.t(), h2)
                h1, h2 = h1[:, None], h2[:, None]
            else:
                Vc = Vk.conj() if is_complex else Vk
                h1 = torch.einsum("knm,nm->km", Vc, W)
                W -= torch.einsum("knm,km->nm", Vk, h1)
                h2 = torch.einsum("knm,nm->km", Vc, W)
                W -= torch.einsum("knm,km->nm", Vk, h2)
            H[:k + 1, k] = (h1 + h2).cpu().numpy()
            hn = cnorm(W)
            H[k + 1, k] = hn
            V[k + 1] = W * torch.as_tensor(np.where(hn > 0, 1.0 / np.maximum(hn, 1e-300), 0.0),
                                           device=B.device, dtype=W.real.dtype if is_complex else W.dtype)
            # Givens rotations per column
            for c in range(m):
                for j in range(k):
                    a0, a1 = H[j, k, c], H[j + 1, k, c]
                    H[j, k, c] = cs[j, c] * a0 + sn[j, c] * a1
                    H[j + 1, k, c] = -np.conj(sn[j, c]) * a0 + cs[j, c] * a1
                cc, ss = _givens(H[k, k, c], H[k + 1, k, c])
                cs[k, c], sn[k, c] = cc, ss
                H[k, k, c] = cc * H[k, k, c] + ss * H[k + 1, k, c]
                H[k + 1, k, c] = 0
                g[k + 1, c] = -np.conj(ss) * g[k, c]
                g[k, c] = cc * g[k, c]
            k_used = k + 1
            est = np.abs(g[k + 1]) / bnorm
            est[done] = 0.0
            history.append(est.copy())
            if (est <= tol).all() or iters >= maxiter:
                break
        # x += V y, y from the triangular system, per column (finished columns keep x)
        Y = np.zeros((k_used, m), hdt)
        for c in range(m):
            if done[c]:
                continue
            Rm = H[:k_used, :k_used, c]
            Y[:, c] = np.linalg.solve(np.triu(Rm), g[:k_used, c])
        Yd = torch.as_tensor(Y, device=B.device, dtype=B.dtype)
        X += torch.einsum("knm,km->nm", V[:k_used], Yd)
    R = B - A(X)
    res = cnorm(R) / bnorm
    out = X.reshape(bd.shape)
    if on_host:
        out = out.cpu()
        if not is_torch:
            out = out.numpy()
    return GmresResult(x=out, iterations=iters, residuals=res, converged=res <= tol * 1.01,
                       history=history)
