"""Track B (3D octree, Helmholtz, complex operators) on the GPU: products/s of
BASELINE's configs in 3D and the accuracy against the O(N^2) Helmholtz sum.

    python tools/track_b.py [--configs C1,C2,C3] [--reps 100] [--dense-max 20000]

Per config and precision (c64 = float32 engine, c128 = float64 engine): us per
product (CUDA events around `reps` back-to-back products, device-resident),
near-field entries, rel. L2 against the serial oracle (mvp_serial on the same
operators) and, up to --dense-max points, against the exact sum.
"""
import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

CONFIGS = {"C1": ("sphere", 2000, 0, 32, 24), "C2": ("sphere", 20000, 1, 32, 32),
           "C3": ("ellipsoid-plates", 200000, 2, 48, 48),
           "C4": ("ellipsoid-plates", 2000000, 3, 64, 64)}   # timing only (no host oracle at 2M)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3")
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--dense-max", type=int, default=20000)
    ap.add_argument("--no-oracle", action="store_true")
    a = ap.parse_args()
    import numpy as np
    import torch
    from oracle.mvp_oracle import mvp_serial, rel_l2
    from paper_1801_03589_b200 import helmholtz as hz
    from paper_1801_03589_b200.plan3 import HelmholtzPlan
    for name in a.configs.split(","):
        kind, n, seed, P, Q = CONFIGS[name]
        t0 = time.perf_counter()
        pts, tree, params, q = hz.track_b_problem(kind, n, seed, P, Q)
        tables = hz.build_tables3(tree, params)
        t_build = time.perf_counter() - t0
        ref = None
        if not a.no_oracle and n <= 200000:
            ref = mvp_serial(tree, hz.build_all3(tree, params, tables), q)
        dense = hz.dense_helmholtz(pts, q, params.k) if n <= a.dense_max else None
        variants = (("c64", True), ("c128", True), ("c64", False)) if n <= 200000 else (("c64", True),)
        for dt, cn in variants:
            t1 = time.perf_counter()
            plan = HelmholtzPlan(tree, tables, dt, complex_near=cn)
            t_plan = time.perf_counter() - t1
            cq = np.complex64 if dt == "c64" else np.complex128
            qd = torch.from_numpy(q.astype(cq)).cuda()
            out = plan.matvec(qd)
            for _ in range(5):
                plan.matvec(qd)
            xr = torch.view_as_real(qd.reshape(n, 1)).permute(0, 2, 1).contiguous()
            yr = torch.empty_like(xr)
            st = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.reps):
                plan.matvec_ptr(xr.data_ptr(), yr.data_ptr(), 1, False, stream=st.cuda_stream)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / a.reps
            phi = out.cpu().numpy()
            rec = {"config": name, "surface": kind, "N": n, "P": P, "Q": Q, "k": round(params.k, 4),
                   "levels": tree.L - tree.l0 + 1, "leaves": tree.n_leaves, "dtype": dt,
                   "near": "complex row-split" if cn else "real 2x2 embedding",
                   "us_per_product": round(us, 1), "products_per_s": round(1e6 / us, 1),
                   "near_entries_complex": plan.stat("near_entries") // (2 if cn else 4),
                   "near_bytes": plan.stat("near_entries") * (4 if dt == "c64" else 8),
                   "kernels": plan.stat("kernels_per_matvec"),
                   "rel_l2_vs_oracle": None if ref is None else float(f"{rel_l2(phi, ref):.3e}"),
                   "rel_l2_vs_dense": None if dense is None else float(f"{rel_l2(phi, dense):.3e}"),
                   "host_tables_s": round(t_build, 2), "plan_s": round(t_plan, 2)}
            print(json.dumps(rec), flush=True)
            plan.close()


if __name__ == "__main__":
    main()
