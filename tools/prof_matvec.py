"""Run K products of the bench workload (for ncu launch lists / captures).

    python tools/prof_matvec.py [--n 2000000] [--k 3] [--dtype f32]
"""
import argparse
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--k", type=int, default=3)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--geometry", default="ellipse-plates")
    ap.add_argument("--P", type=int, default=64)
    ap.add_argument("--Q", type=int, default=64)
    a = ap.parse_args()
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.plan import NesaPlan
    pts = nesa.generate_sources(nesa.CurveSpec(kind=a.geometry, seed=3), a.n)
    tree = nesa.build_tree(pts, nesa.TreeParams(P=a.P))
    tables = nesa.build_tables(tree, nesa.NesaParams(Q=a.Q))
    plan = NesaPlan(tree, tables, dtype=a.dtype)
    cdt = np.complex64 if a.dtype == "f32" else np.complex128
    q = torch.from_numpy(nesa.random_rhs(a.n, 3).astype(cdt)).cuda()
    phi = torch.empty_like(q)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(a.k):
        plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, stream=s)
    torch.cuda.synchronize()
    print("ok", float(phi.abs().sum()))


if __name__ == "__main__":
    main()
