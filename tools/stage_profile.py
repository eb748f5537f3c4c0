"""Stage durations inside the concurrent product (profiled graph events).

    python tools/stage_profile.py [--n 2000000] [--reps 100]

near: the near-field kernel (stream s1); far: radiation .. downward pass
(stream s0, concurrent with near); reception; total.  Medians in us.
"""
import argparse
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--reps", type=int, default=100)
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.plan import NesaPlan
    pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=3), a.n)
    tree = nesa.build_tree(pts, nesa.TreeParams(P=64))
    plan = NesaPlan(tree, nesa.build_tables(tree, nesa.NesaParams(Q=64)), dtype="f32")
    q = torch.from_numpy(nesa.random_rhs(a.n, 3).astype(np.complex64)).cuda()
    phi = torch.empty_like(q)
    st = torch.cuda.current_stream()
    for _ in range(10):
        plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, stream=st.cuda_stream, profile=True)
    plan.profile_reset()
    for _ in range(a.reps):
        plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, stream=st.cuda_stream, profile=True)
    torch.cuda.synchronize()
    for stg in ("total", "near", "far", "reception"):
        print(f"{stg:10s} {np.median(plan.profile_read(stg)) * 1e3:8.1f} us")


if __name__ == "__main__":
    main()
