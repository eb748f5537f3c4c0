"""Randomised parity sweep of the GPU product against the oracle.

    python tools/parity_sweep.py [--cases 40] [--seed 0]

Each case draws a geometry (the reference's wave curve, a random circle, the
ellipse + plates analog), N (2k-40k), leaf P, Q (6-96), precision, vector
width (1-5 real or 1-2 complex columns), near / far flags and a forced
wide-level threshold, builds the plan (device assembly, or the host
OperatorSet route), and compares with oracle/mvp_oracle.mvp_serial:
float64 <= 1e-12, float32 <= 1e-5 (relative L2).  Prints one line per case
and the failures at the end; exit status 1 if any case fails.
"""
import argparse
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
c = json.loads(sys.argv[2])
import torch
import paper_1801_03589_b200 as nesa
from oracle.mvp_oracle import mvp_serial, rel_l2
spec = nesa.CurveSpec(kind=c["geo"], seed=c["seed"]) if c["geo"] != "wave" else nesa.CurveSpec()
pts = nesa.generate_sources(spec, c["n"])
tree = nesa.build_tree(pts, nesa.TreeParams(P=c["P"]))
params = nesa.NesaParams(Q=c["Q"])
ops = nesa.build_all(tree, params)
rng = np.random.default_rng(c["seed"])
shape = (c["n"],) if c["cols"] == 1 else (c["n"], c["cols"])
q = rng.standard_normal(shape)
if c["cplx"]:
    q = q + 1j * rng.standard_normal(shape)
ref = mvp_serial(tree, ops, q, near=c["near"], far=c["far"])
qq = q if c["dt"] == "f64" else q.astype(np.complex64 if c["cplx"] else np.float32)
phi = nesa.mvp(tree, ops if c["opset"] else params, qq, near=c["near"], far=c["far"])
print(json.dumps({"err": rel_l2(phi, ref)}))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=40)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    import json
    import random
    rnd = random.Random(a.seed)
    fails = []
    for i in range(a.cases):
        c = {"geo": rnd.choice(["wave", "circle-random", "ellipse-plates"]),
             "n": rnd.choice([2000, 6000, 15000, 40000]), "seed": rnd.randrange(100),
             "P": rnd.choice([16, 32, 48, 64]), "Q": rnd.choice([6, 10, 16, 24, 32, 48, 64, 96]),
             "dt": rnd.choice(["f32", "f64"]), "cplx": rnd.random() < 0.5,
             "near": True, "far": True, "opset": rnd.random() < 0.25,
             "wide": rnd.choice([None, None, "64", "256"])}
        c["cols"] = rnd.choice([1, 1, 2]) if c["cplx"] else rnd.choice([1, 1, 2, 3, 5])
        flags = rnd.random()
        if flags < 0.15:
            c["near"] = False
        elif flags < 0.3:
            c["far"] = False
        env = dict(os.environ)
        if c["wide"]:
            env["NESA_WIDE_LEVEL"] = c["wide"]
        p = subprocess.run([sys.executable, "-c", CHILD, HERE, json.dumps(c)], env=env, capture_output=True,
                           text=True, timeout=900)
        line = [x for x in p.stdout.splitlines() if x.startswith("{")]
        tol = 1e-12 if c["dt"] == "f64" else 1e-5
        if not line:
            err, ok = None, False
            msg = p.stderr.strip().splitlines()[-1] if p.stderr.strip() else "no output"
        else:
            err = json.loads(line[-1])["err"]
            ok = err <= tol
            msg = ""
        print(i, "ok " if ok else "BAD", c, err, msg, flush=True)
        if not ok:
            fails.append((c, err, msg))
    print(f"{len(fails)} of {a.cases} cases failed")
    for f in fails:
        print("FAIL", f)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
