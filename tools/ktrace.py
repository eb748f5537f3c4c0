"""Concurrent kernel timeline of one product from in-kernel %globaltimer
records (no graph nodes added, schedule unperturbed).

    python tools/ktrace.py [--n 2000000] [--reps 5] [--chrome out.json]

Per kernel launch (tag, grid): first CTA start, last CTA end (us from the
product's first CTA), span, CTA count; medians over reps.
"""
import argparse
import ctypes
import json
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

TAGS = {2: "scatter", 3: "gather (original order)", 10: "blockgemv(store: near)", 11: "blockgemv(scatter: U)",
        30: "fused_up", 31: "fused_down", 33: "reduce", 40: "tgemm",
        41: "tgemm_wt (FFMA)", 43: "tgemm_tc2 (tcgen05, A in TMEM)", 44: "tgemm_tc3 (fine units)", 45: "tgemm_tc3 (coarse units)", 50: "level_wt up-leaf",
        51: "level_wt up-sum", 52: "level_wt down", 54: "level_wt down + beta (leaf)", 60: "radiation moments (in-kernel A)", 62: "radiation (tcgen05 moment map)",
        70: "reception series", 71: "reception series (beta in)", 72: "reception series (float64)", 80: "level_tc up-leaf", 81: "level_tc up-sum",
        82: "level_tc down", 84: "level_tc down + beta (leaf)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--chrome", default="")
    ap.add_argument("--near", type=int, default=1)
    ap.add_argument("--far", type=int, default=1)
    ap.add_argument("--dtype", default="f32", help="f32 (complex64) or f64 (complex128)")
    ap.add_argument("--world", type=int, default=1, help="trace rank --rank's sub-plan of this partition")
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--P", type=int, default=64)
    ap.add_argument("--Q", type=int, default=64)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--ends", type=int, default=0, help="print the distribution of CTA end times of this kernel tag")
    ap.add_argument("--split", action="store_true",
                    help="separate repeated launches of one (kernel, grid): CTA records in start order, grid at a time")
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.plan import NesaPlan
    pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=a.seed), a.n)
    tree = nesa.build_tree(pts, nesa.TreeParams(P=a.P))
    lr = None
    if a.world > 1:
        from paper_1801_03589_b200.dist import partition_leaves
        lr = partition_leaves(tree, a.world, a.Q)[a.rank]
    plan = NesaPlan(tree, nesa.build_tables(tree, nesa.NesaParams(Q=a.Q)), dtype=a.dtype, leaf_range=lr)
    cdt = np.complex64 if a.dtype == "f32" else np.complex128
    q = torch.from_numpy(nesa.random_rhs(a.n, a.seed).astype(cdt)).cuda()
    phi = torch.empty_like(q)
    st = torch.cuda.current_stream()
    lib = plan.lib
    cap = 1 << 16
    for _ in range(5):
        plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, near=bool(a.near), far=bool(a.far),
                        stream=st.cuda_stream)
    lib.nesa_ktrace_enable(plan.handle, cap)
    buf = (ctypes.c_uint64 * (4 * cap))()
    runs = []
    for _ in range(a.reps):
        plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, near=bool(a.near), far=bool(a.far),
                        stream=st.cuda_stream)
        torch.cuda.synchronize()
        n = lib.nesa_ktrace_read(plan.handle, buf, cap)
        rec = np.frombuffer(buf, dtype=np.uint64, count=4 * n).reshape(n, 4).astype(np.int64)
        t0 = rec[:, 2].min()
        if a.ends:
            e = np.sort(rec[rec[:, 0] == a.ends, 3] - t0) / 1e3
            if len(e):
                print(f"tag {a.ends}: CTA end times (us) min {e[0]:.1f} p10 {e[len(e)//10]:.1f} "
                      f"p50 {e[len(e)//2]:.1f} p90 {e[len(e)*9//10]:.1f} max {e[-1]:.1f} (n={len(e)})")
        launches = {}
        if a.split:
            # launch index of each record: rank of its start among the records of its (tag, grid), // grid
            order = np.lexsort((rec[:, 2], rec[:, 1], rec[:, 0]))
            rec = rec[order]
            sub = np.zeros(len(rec), dtype=np.int64)
            i = 0
            while i < len(rec):
                j = i
                while j < len(rec) and rec[j, 0] == rec[i, 0] and rec[j, 1] == rec[i, 1]:
                    j += 1
                sub[i:j] = np.arange(j - i) // max(1, int(rec[i, 1]))
                i = j
        else:
            sub = np.zeros(len(rec), dtype=np.int64)
        for (tag, grid, s, e), sb in zip(rec, sub):
            k = (int(tag), int(grid), int(sb))
            lo, hi, c = launches.get(k, (1 << 62, 0, 0))
            launches[k] = (min(lo, s - t0), max(hi, e - t0), c + 1)
        runs.append(launches)
    lib.nesa_ktrace_enable(plan.handle, 0)
    keys = sorted(runs[0], key=lambda k: runs[0][k][0])
    rows = []
    print(f"{'kernel':34s} {'grid':>6s} {'start':>8s} {'end':>8s} {'span':>8s} {'CTAs':>6s}")
    for k in keys:
        st_ = np.median([r[k][0] for r in runs if k in r]) / 1e3
        en = np.median([r[k][1] for r in runs if k in r]) / 1e3
        c = runs[0][k][2]
        name = TAGS.get(k[0], str(k[0]))
        rows.append((name, k[1], st_, en))
        print(f"{name:34s} {k[1]:6d} {st_:8.1f} {en:8.1f} {en - st_:8.1f} {c:6d}")
    tot = np.median([max(v[1] for v in r.values()) for r in runs]) / 1e3
    print(f"product span (first CTA start -> last CTA end): {tot:.1f} us")
    if a.chrome:
        ev = [{"name": n, "ph": "X", "ts": s, "dur": e - s, "pid": 0,
               "tid": 1 if n.startswith("blockgemv") else 0, "args": {"grid": g}}
              for n, g, s, e in rows]
        json.dump({"traceEvents": ev}, open(a.chrome, "w"))


if __name__ == "__main__":
    main()
