"""One Track B product (3D ellipsoid + plates, Helmholtz, complex64) for ncu.

    python tools/track_b_profile.py [--n 2000000] [--P 64] [--Q 64] [--k 2]
"""
import argparse
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--P", type=int, default=64)
    ap.add_argument("--Q", type=int, default=64)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--k", type=int, default=2)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_1801_03589_b200 import helmholtz as hz
    from paper_1801_03589_b200.plan3 import HelmholtzPlan
    pts, tree, params, q = hz.track_b_problem("ellipsoid-plates", a.n, a.seed, a.P, a.Q)
    plan = HelmholtzPlan(tree, hz.build_tables3(tree, params), "c64")
    qd = torch.from_numpy(q.astype(np.complex64)).cuda()
    for _ in range(a.k):
        plan.matvec(qd)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
