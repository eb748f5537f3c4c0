"""Products/s on the BASELINE configurations C1-C4 (2D analogs).

    python tools/configs.py [--reps 200]

C1: unit circle (random angles, seed 0), N = 2 000,   P = 32, Q = 24
C2: unit circle (seed 1),                N = 20 000,  P = 32, Q = 32
C3: ellipse (5, 0.5) + 2 plates, seed 2, N = 200 000, P = 48, Q = 48
C4: ellipse (5, 0.5) + 2 plates, seed 3, N = 2M,      P = 64, Q = 64
Each with a float32 plan / complex64 vector and a float64 plan / complex128
vector; device-resident, CUDA events around `reps` back-to-back products.
C5 (--c5): ellipse + plates, seed 4, N = 200 000, 64 plane waves
exp(-j k d_m . r) (k at 10 points per wavelength), Q in {24, 48, 96} x leaf
P in {32, 64, 128}, complex64: one product of all 64 right-hand sides.
"""
import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

CONFIGS = [
    ("C1", "circle-random", 2_000, 0, 32, 24),
    ("C2", "circle-random", 20_000, 1, 32, 32),
    ("C3", "ellipse-plates", 200_000, 2, 48, 48),
    ("C4", "ellipse-plates", 2_000_000, 3, 64, 64),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--only", default="")
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--gemm-only", action="store_true", help="C5: time only the GEMM far-field path")
    a = ap.parse_args()
    if a.c5:
        return c5(a)
    import numpy as np
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.plan import NesaPlan
    out = []
    for name, kind, n, seed, P, Q in CONFIGS:
        if a.only and name not in a.only.split(","):
            continue
        t0 = time.perf_counter()
        pts = nesa.generate_sources(nesa.CurveSpec(kind=kind, seed=seed), n)
        tree = nesa.build_tree(pts, nesa.TreeParams(P=P))
        tables = nesa.build_tables(tree, nesa.NesaParams(Q=Q))
        t_build = time.perf_counter() - t0
        q = nesa.random_rhs(n, seed)
        for dt, cdt in (("f32", np.complex64), ("f64", np.complex128)):
            plan = NesaPlan(tree, tables, dtype=dt)
            qd = torch.from_numpy(q.astype(cdt)).cuda()
            phi = torch.empty_like(qd)
            st = torch.cuda.current_stream()
            for _ in range(10):
                plan.matvec_ptr(qd.data_ptr(), phi.data_ptr(), 1, True, stream=st.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(a.reps):
                plan.matvec_ptr(qd.data_ptr(), phi.data_ptr(), 1, True, stream=st.cuda_stream)
            e1.record(st)
            e1.synchronize()
            us = e0.elapsed_time(e1) / a.reps * 1e3
            rec = {"config": name, "N": n, "P": P, "Q": Q, "levels": tree.L - tree.l0 + 1,
                   "plan": dt, "us_per_product": round(us, 1), "products_per_s": round(1e6 / us, 1),
                   "kernels": plan.stat("kernels_per_matvec"), "host_build_s": round(t_build, 2)}
            print(json.dumps(rec), flush=True)
            out.append(rec)
            plan.close()
    return out


def c5(a):
    import numpy as np
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.fastmvp import RhsLanes
    from paper_1801_03589_b200.plan import NesaPlan
    n = 200_000
    spec = nesa.CurveSpec(kind="ellipse-plates", seed=4)
    pts = nesa.generate_sources(spec, n)
    k = nesa.wavenumber(spec, n)
    q = nesa.plane_wave_rhs(pts, k, 64).astype(np.complex64)
    qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    phi = torch.empty_like(qd)
    st = torch.cuda.current_stream()
    for P in (32, 64, 128):
        tree = nesa.build_tree(pts, nesa.TreeParams(P=P))
        for Q in (24, 48, 96):
            plan = NesaPlan(tree, nesa.build_tables(tree, nesa.NesaParams(Q=Q)), dtype="f32")
            rec = {"config": "C5", "N": n, "P": P, "Q": Q, "rhs": 64, "levels": tree.L - tree.l0 + 1,
                   "plan": "f32"}
            lanes = RhsLanes(plan, 4)
            lanes8 = RhsLanes(plan, 8)
            # stored V / U: the far field as batched GEMMs over the 128 columns
            gplan = NesaPlan(tree, nesa.build_tables(tree, nesa.NesaParams(Q=Q)), dtype="f32",
                             stored_vu=True)
            assert gplan.stat("far_wide") == 1
            engines = [("gemm", gplan)] + ([] if a.gemm_only else
                                            [("one_plan", plan), ("lanes4", lanes), ("lanes8", lanes8)])
            for tag, eng in engines:
                for _ in range(3):
                    eng.matvec_ptr(qd.data_ptr(), phi.data_ptr(), 64, True, stream=st.cuda_stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = max(3, a.reps // 20)
                e0.record(st)
                for _ in range(reps):
                    eng.matvec_ptr(qd.data_ptr(), phi.data_ptr(), 64, True, stream=st.cuda_stream)
                e1.record(st)
                e1.synchronize()
                ms = e0.elapsed_time(e1) / reps
                rec[f"ms_per_64rhs_product_{tag}"] = round(ms, 3)
                rec[f"rhs_products_per_s_{tag}"] = round(64e3 / ms, 1)
            # the near field alone: one tcgen05 GEMM pass over the 128 real columns
            if plan.stat("near_wide"):
                for _ in range(3):
                    plan.near_wide_ptr(qd.data_ptr(), phi.data_ptr(), 128, 0, 128, stream=st.cuda_stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(20):
                    plan.near_wide_ptr(qd.data_ptr(), phi.data_ptr(), 128, 0, 128, stream=st.cuda_stream)
                e1.record(st)
                e1.synchronize()
                rec["near_wide_ms"] = round(e0.elapsed_time(e1) / 20, 4)
                rec["near_entries"] = plan.stat("near_entries")
            print(json.dumps(rec), flush=True)
            for p_ in lanes.plans[1:] + lanes8.plans[1:]:
                p_.close()
            plan.close()
            gplan.close()


if __name__ == "__main__":
    main()
