"""GMRES on the benchmark problem: (shift I + K~) x = b at N = 2M, complex64.

    python tools/solve_c4.py [--n 2000000] [--shift 200] [--tol 1e-5] [--nrhs 1]

Prints iterations, wall time, time per iteration and the final relative
residual (recomputed with one more GPU product).
"""
import argparse
import os
import sys
import time

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--shift", type=float, default=200.0)
    ap.add_argument("--tol", type=float, default=1e-5)
    ap.add_argument("--nrhs", type=int, default=1)
    ap.add_argument("--restart", type=int, default=30)
    ap.add_argument("--orth", default="auto", help="auto (fused device CGS2) | torch")
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_1801_03589_b200 as nesa
    pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=3), a.n)
    tree = nesa.build_tree(pts, nesa.TreeParams(P=64))
    tables = nesa.build_tables(tree, nesa.NesaParams(Q=64))
    rng = np.random.default_rng(3)
    b = (rng.standard_normal((a.n, a.nrhs)) + 1j * rng.standard_normal((a.n, a.nrhs))).astype(np.complex64)
    bd = torch.from_numpy(b if a.nrhs > 1 else b[:, 0].copy()).cuda()
    nesa.gmres(tree, tables, bd, shift=a.shift, tol=1e-1, restart=2, maxiter=2)  # plan + graphs
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = nesa.gmres(tree, tables, bd, shift=a.shift, tol=a.tol, restart=a.restart, maxiter=1000,
                     orthogonalise=a.orth)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"N={a.n} nrhs={a.nrhs} shift={a.shift} orth={a.orth} iterations={res.iterations} "
          f"time={dt:.3f}s per_iteration={1e3 * dt / max(res.iterations, 1):.3f}ms "
          f"residual={res.residuals} converged={res.converged}")


if __name__ == "__main__":
    main()
