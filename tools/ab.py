"""A/B timing of library builds on the bench workload (C4 product).

    python tools/ab.py ab/libA.so ab/libB.so [--rounds 3] [--steps 200]
    python tools/ab.py lib.so lib.so:NESA_U_TERMS=22     (a spec may add environment settings)
    python tools/ab.py lib.so lib.so:AB_PROFILE=1        (with the near-field event nodes bench.py times)
    python tools/ab.py a.so:AB_CFG=200000/48/48/2,AB_DTYPE=f64 b.so:AB_CFG=200000/48/48/2,AB_DTYPE=f64   (C3, float64 plan)

Each round runs every library in a fresh process (NESA_LIB selects it),
alternating the order, and times `steps` back-to-back products with CUDA
events after a warm-up; prints the per-library median of the rounds.
"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, json, numpy as np, torch
sys.path.insert(0, sys.argv[1])
prof = "near" if os.environ.get("AB_PROFILE") else False
import paper_1801_03589_b200 as nesa
from paper_1801_03589_b200.plan import NesaPlan
steps = int(sys.argv[2])
# AB_CFG=N,P,Q,seed (default the C4 bench workload), AB_DTYPE=f32|f64
N, PP, QQ, SEED = (int(x) for x in os.environ.get("AB_CFG", "2000000/64/64/3").split("/"))
dt = os.environ.get("AB_DTYPE", "f32")
pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=SEED), N)
tree = nesa.build_tree(pts, nesa.TreeParams(P=PP))
plan = NesaPlan(tree, nesa.build_tables(tree, nesa.NesaParams(Q=QQ)), dtype=dt)
q = torch.from_numpy(nesa.random_rhs(N, SEED).astype(np.complex64 if dt == "f32" else np.complex128)).cuda()
phi = torch.empty_like(q)
bufs = [(q, phi)]
if os.environ.get("AB_ALT"):  # two buffer pairs, alternating (the io nodes re-pointed every launch)
    bufs.append((q.clone(), torch.empty_like(q)))
st = torch.cuda.current_stream()
for i in range(20):
    qq, pp = bufs[i % len(bufs)]
    plan.matvec_ptr(qq.data_ptr(), pp.data_ptr(), 1, True, stream=st.cuda_stream, profile=prof)
torch.cuda.synchronize()
res = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(steps):
        qq, pp = bufs[i % len(bufs)]
        plan.matvec_ptr(qq.data_ptr(), pp.data_ptr(), 1, True, stream=st.cuda_stream, profile=prof)
    e1.record(st)
    e1.synchronize()
    res.append(e0.elapsed_time(e1) / steps)
print(json.dumps({"ms": min(res)}))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    out = {lib: [] for lib in a.libs}
    for r in range(a.rounds):
        order = a.libs if r % 2 == 0 else list(reversed(a.libs))
        for lib in order:
            path, _, extra = lib.partition(":")
            env = dict(os.environ, NESA_LIB=os.path.abspath(path))
            for kv in filter(None, extra.split(",")):
                k, _, v = kv.partition("=")
                env[k] = v
            p = subprocess.run([sys.executable, "-c", CHILD, HERE, str(a.steps)], env=env,
                               capture_output=True, text=True)
            line = [x for x in p.stdout.splitlines() if x.startswith("{")]
            if not line:
                print(lib, "failed", p.stderr[-800:])
                continue
            out[lib].append(json.loads(line[-1])["ms"])
            print(lib, f"{out[lib][-1] * 1e3:.1f} us", flush=True)
    import statistics
    for lib, v in out.items():
        if v:
            print(f"{lib}: median {statistics.median(v) * 1e3:.1f} us  all {[round(x * 1e3, 1) for x in v]}")


if __name__ == "__main__":
    main()
