"""Time the bench product under several NESA_* environment settings in one
process (the tree and tables are built once; each setting gets its own plan).

    python tools/sweep.py "" "NESA_WIDE_LEVEL=1024" "NESA_U_TERMS=22;NESA_V_MOMENTS=32" ...

Per setting: median / min us per product over --reps blocks of --k graph
launches (CUDA events on the launch stream), and whether phi is bitwise equal
to the first setting's.  With --ktrace, also the per-kernel timeline.
"""
import argparse
import ctypes
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

from tools.ktrace import TAGS  # noqa: E402


NEAR = FAR = True


def timeline(plan, q, phi, st, reps=3):
    import numpy as np
    import torch
    lib = plan.lib
    cap = 1 << 16
    lib.nesa_ktrace_enable(plan.handle, cap)
    buf = (ctypes.c_uint64 * (4 * cap))()
    runs = []
    for _ in range(reps):
        plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, near=NEAR, far=FAR, stream=st.cuda_stream)
        torch.cuda.synchronize()
        n = lib.nesa_ktrace_read(plan.handle, buf, cap)
        rec = np.frombuffer(buf, dtype=np.uint64, count=4 * n).reshape(n, 4).astype(np.int64)
        t0 = rec[:, 2].min()
        launches = {}
        for tag, grid, s, e in rec:
            k = (int(tag), int(grid))
            lo, hi, c = launches.get(k, (1 << 62, 0, 0))
            launches[k] = (min(lo, s - t0), max(hi, e - t0), c + 1)
        runs.append(launches)
    lib.nesa_ktrace_enable(plan.handle, 0)
    keys = sorted(runs[0], key=lambda k: runs[0][k][0])
    for k in keys:
        s_ = np.median([r[k][0] for r in runs if k in r]) / 1e3
        e_ = np.median([r[k][1] for r in runs if k in r]) / 1e3
        print(f"    {TAGS.get(k[0], str(k[0])):34s} {k[1]:6d} {s_:8.1f} {e_:8.1f} {e_ - s_:8.1f}")
    tot = np.median([max(v[1] for v in r.values()) for r in runs]) / 1e3
    print(f"    span {tot:.1f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("settings", nargs="*", default=[""])
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ktrace", action="store_true")
    ap.add_argument("--near", type=int, default=1)
    ap.add_argument("--far", type=int, default=1)
    a = ap.parse_args()
    global NEAR, FAR
    NEAR, FAR = bool(a.near), bool(a.far)
    import numpy as np
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.plan import NesaPlan
    pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=3), a.n)
    tree = nesa.build_tree(pts, nesa.TreeParams(P=64))
    tables = nesa.build_tables(tree, nesa.NesaParams(Q=64))
    q = torch.from_numpy(nesa.random_rhs(a.n, 3).astype(np.complex64)).cuda()
    st = torch.cuda.current_stream()
    ref = None
    base_env = dict(os.environ)
    for setting in a.settings:
        os.environ.clear()
        os.environ.update(base_env)
        for kv in filter(None, setting.split(";")):
            k, v = kv.split("=", 1)
            os.environ[k] = v
        plan = NesaPlan(tree, tables, dtype="f32")
        phi = torch.empty_like(q)
        for _ in range(20):
            plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, near=NEAR, far=FAR, stream=st.cuda_stream)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(a.k):
                plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, near=NEAR, far=FAR, stream=st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / a.k)
        out = phi.cpu().numpy()
        if ref is None:
            ref = out
            same = "ref"
        else:
            same = "bitwise" if np.array_equal(out, ref) else \
                f"DIFF rel {np.linalg.norm(out - ref) / np.linalg.norm(ref):.2e}"
        print(f"[{setting or 'default'}] median {np.median(ts):.1f} us  min {min(ts):.1f} us  {same}",
              flush=True)
        if a.ktrace:
            timeline(plan, q, phi, st)
        plan.close()
        del plan
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
