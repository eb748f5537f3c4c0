"""Per-kernel timeline of one profiled product of the bench workload.

    NESA_TRACE=1 python tools/trace.py [--n 2000000] [--reps 20]

Prints, for each kernel, the median (over reps) time of the event recorded
after it, in microseconds from the product's start, and the gap to the
previous event on the same stream.  Event nodes break programmatic
dependent launch between kernels, so the total is a little longer than the
untraced product.
"""
import argparse
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def main():
    os.environ.setdefault("NESA_TRACE", "1")
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--near", type=int, default=1)
    ap.add_argument("--far", type=int, default=1)
    ap.add_argument("--chrome", default="", help="also write a Chrome trace (chrome://tracing) here")
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.plan import NesaPlan
    pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=3), a.n)
    tree = nesa.build_tree(pts, nesa.TreeParams(P=64))
    tables = nesa.build_tables(tree, nesa.NesaParams(Q=64))
    plan = NesaPlan(tree, tables, dtype="f32")
    q = torch.from_numpy(nesa.random_rhs(a.n, 3).astype(np.complex64)).cuda()
    phi = torch.empty_like(q)
    st = torch.cuda.current_stream()
    runs = []
    for i in range(a.reps + 5):
        plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, near=bool(a.near), far=bool(a.far),
                        stream=st.cuda_stream, profile=True)
        torch.cuda.synchronize()
        if i >= 5:
            runs.append(plan.trace_read())
    names = [n for n, _ in runs[0]]
    t = np.median(np.array([[v for _, v in r] for r in runs]), axis=0) * 1e3
    last = {}
    for n, v in zip(names, t):
        stream = "s1" if n.startswith("near") else "s0"
        prev = last.get(stream, 0.0)
        print(f"{n:12s} {v:8.1f} us   +{v - prev:7.1f}")
        last[stream] = v
    tot = plan.profile_read("total")
    print(f"total (median) {np.median(tot) * 1e3:.1f} us")
    if a.chrome:
        # one complete event per kernel: from the previous event on its stream
        import json
        ev, last = [], {}
        for n, v in zip(names, t):
            stream = "s1" if n.startswith("near") else "s0"
            t0 = last.get(stream, 0.0)
            ev.append({"name": n, "ph": "X", "ts": t0, "dur": max(v - t0, 0.0), "pid": 0,
                       "tid": 1 if stream == "s1" else 0})
            last[stream] = v
        json.dump({"traceEvents": ev, "displayTimeUnit": "ns"}, open(a.chrome, "w"))


if __name__ == "__main__":
    main()
