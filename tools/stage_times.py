"""Time near-only / far-only / full products of the bench workload (CUDA events).

    python tools/stage_times.py [--n 2000000] [--reps 100]
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
    ap.add_argument("--dtype", default="f32")
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.plan import NesaPlan
    pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=3), a.n)
    tree = nesa.build_tree(pts, nesa.TreeParams(P=64))
    tables = nesa.build_tables(tree, nesa.NesaParams(Q=64))
    plan = NesaPlan(tree, tables, dtype=a.dtype)
    cdt = np.complex64 if a.dtype == "f32" else np.complex128
    q = torch.from_numpy(nesa.random_rhs(a.n, 3).astype(cdt)).cuda()
    phi = torch.empty_like(q)
    st = torch.cuda.current_stream()
    for name, near, far, prof in (("full", True, True, False), ("full+prof", True, True, True),
                                  ("near", True, False, False), ("far", False, True, False)):
        for _ in range(10):
            plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, near=near, far=far,
                            stream=st.cuda_stream, profile=prof)
        if prof:
            plan.profile_reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(a.reps):
            plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, near=near, far=far,
                            stream=st.cuda_stream, profile=prof)
        e1.record(st)
        e1.synchronize()
        print(f"{name:9s} {e0.elapsed_time(e1) / a.reps * 1e3:8.1f} us  "
              f"(NESA_WIDE_LEVEL={os.environ.get('NESA_WIDE_LEVEL', '2048')})")


if __name__ == "__main__":
    main()
