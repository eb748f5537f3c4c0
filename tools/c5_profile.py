"""One C5 64-RHS product on the GEMM far-field path (for ncu launch lists).

    python tools/c5_profile.py [--P 64] [--Q 48] [--k 2]
"""
import argparse
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=64)
    ap.add_argument("--Q", type=int, default=48)
    ap.add_argument("--k", type=int, default=2)
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.plan import NesaPlan
    n = 200_000
    spec = nesa.CurveSpec(kind="ellipse-plates", seed=4)
    pts = nesa.generate_sources(spec, n)
    q = nesa.plane_wave_rhs(pts, nesa.wavenumber(spec, n), 64).astype(np.complex64)
    qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    phi = torch.empty_like(qd)
    tree = nesa.build_tree(pts, nesa.TreeParams(P=a.P))
    plan = NesaPlan(tree, nesa.build_tables(tree, nesa.NesaParams(Q=a.Q)), dtype="f32", stored_vu=True)
    t = tree.arrays
    print("leaves", tree.n_leaves, "groups", t.n_groups, "d_refs", plan.stat("d_refs"),
          "near_entries", plan.stat("near_entries"), flush=True)
    for _ in range(a.k):
        plan.matvec_ptr(qd.data_ptr(), phi.data_ptr(), 64, True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
