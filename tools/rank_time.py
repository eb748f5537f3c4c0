"""Per-rank product time of the multi-GPU partition, measured one rank at a
time on one GPU (the halo all_gather is skipped: no NCCL peers here).

    python tools/rank_time.py [--n 2000000] [--worlds 2,4,8]

For each world size: every rank's sub-plan (NesaPlan(leaf_range=...)) runs
stage 1 + stage 2 back to back, or (--one-graph) the single-graph schedule the
distributed plan uses (nesa_plan_create_dist: the near field overlaps the
whole far chain); the max over ranks plus the exchange is the distributed
product time.  This is a projection for DESIGN.md, not a
multi-GPU measurement.
"""
import argparse
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--one-graph", action="store_true",
                    help="the distributed plan's single-graph schedule (near field overlapping the "
                         "whole far chain), exchange omitted; default: stage 1 + stage 2")
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.dist import partition_leaves
    from paper_1801_03589_b200.plan import NesaPlan
    pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=3), a.n)
    tree = nesa.build_tree(pts, nesa.TreeParams(P=64))
    tables = nesa.build_tables(tree, nesa.NesaParams(Q=64))
    q = torch.from_numpy(nesa.random_rhs(a.n, 3).astype(np.complex64)).cuda()
    phi = torch.zeros_like(q)
    st = torch.cuda.current_stream()
    for w in [int(x) for x in a.worlds.split(",")]:
        times = []
        for r, lr in enumerate(partition_leaves(tree, w, 64)):
            plan = NesaPlan(tree, tables, dtype="f32", leaf_range=lr)
            stages = (0,) if a.one_graph else (1, 2)
            run = lambda: [plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True,  # noqa: E731
                                           stream=st.cuda_stream, stage=s) for s in stages]
            for _ in range(5):
                run()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(a.k):
                run()
            e1.record(st)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3 / a.k)
            plan.close()
        mode = "one graph" if a.one_graph else "stage 1 + stage 2"
        print(f"world {w}: per-rank us ({mode}, no exchange) "
              f"{' '.join(f'{t:.0f}' for t in times)}; max {max(times):.0f} us -> "
              f"{1e6 / max(times):.0f} products/s before the exchange", flush=True)


if __name__ == "__main__":
    main()
