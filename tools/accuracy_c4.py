"""Approximation error of the bench product at C4 (N = 2M) against the exact
O(N^2) sum on the GPU (float64, ~4e12 pairs), plus the C1-C3 configurations.

    python tools/accuracy_c4.py [--n 2000000]
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
    a = ap.parse_args()
    import numpy as np
    import paper_1801_03589_b200 as nesa
    cases = [("C1 circle", 2000, 32, 24, "circle", 0), ("C2 circle", 20000, 32, 32, "circle", 1),
             ("C3 ellipse+plates", 200000, 48, 48, "ellipse-plates", 2),
             ("C4 ellipse+plates", a.n, 64, 64, "ellipse-plates", 3)]
    for name, n, P, Q, kind, seed in cases:
        pts = nesa.generate_sources(nesa.CurveSpec(kind=kind, seed=seed), n)
        tree = nesa.build_tree(pts, nesa.TreeParams(P=P))
        tables = nesa.build_tables(tree, nesa.NesaParams(Q=Q))
        q = nesa.random_rhs(n, seed)
        t0 = time.perf_counter()
        ref = nesa.dense_matvec_gpu(pts, q)
        td = time.perf_counter() - t0
        for dt in ("f32", "f64"):
            qq = q.astype(np.complex64 if dt == "f32" else np.complex128)
            phi = nesa.mvp(tree, tables, qq)
            err = np.linalg.norm(phi - ref) / np.linalg.norm(ref)
            print(f"{name:20s} N={n:8d} P={P} Q={Q} {dt}: rel L2 vs exact sum {err:.3e} "
                  f"(exact sum on the GPU: {td:.2f} s)", flush=True)


if __name__ == "__main__":
    main()
