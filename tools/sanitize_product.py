"""One product per precision at a chosen size, for compute-sanitizer runs:

    compute-sanitizer --tool racecheck python tools/sanitize_product.py --n 200000
    compute-sanitizer --tool synccheck python tools/sanitize_product.py --n 200000

Default: BASELINE C3 2D analog (200k points on ellipse + plates, seed 2,
P = 48, Q = 48), complex64 (float32 plan, the bench's kernel mix incl. the
tensor-core translation with --q 64) and complex128.  Exits non-zero if a
product disagrees with the plain GPU run by more than the tolerance.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200000)
    ap.add_argument("--p", type=int, default=48)
    ap.add_argument("--q", type=int, default=48)
    ap.add_argument("--seed", type=int, default=2)
    ap.add_argument("--prec", default="c64,c128")
    a = ap.parse_args()
    import paper_1801_03589_b200 as nesa
    pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=a.seed), a.n)
    tree = nesa.build_tree(pts, nesa.TreeParams(P=a.p))
    params = nesa.NesaParams(Q=a.q)
    q = nesa.random_rhs(a.n, a.seed)
    for prec in a.prec.split(","):
        qq = q.astype(np.complex64) if prec == "c64" else q
        phi = nesa.mvp(tree, params, qq)
        print(prec, "norm", float(np.linalg.norm(phi)), flush=True)


if __name__ == "__main__":
    main()
