"""Real (one-column) float32 products at the Q = 64 bench geometry against the oracle."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1801_03589_b200 as nesa
from paper_1801_03589_b200.plan import NesaPlan
from oracle.mvp_oracle import mvp_serial, rel_l2
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=3), n)
tree = nesa.build_tree(pts, nesa.TreeParams(P=64))
params = nesa.NesaParams(Q=64)
ops = nesa.build_all(tree, params)
q = nesa.random_rhs(n, 3, complex_=False)
ref = mvp_serial(tree, ops, q)
for env in ({}, {"NESA_TC": "0"}):
    for k in ("NESA_TC",):
        os.environ.pop(k, None)
    os.environ.update(env)
    plan = NesaPlan(tree, params, dtype="f32")
    qd = torch.from_numpy(q.astype(np.float32)).cuda(); ph = torch.empty_like(qd)
    for near, far in ((True, True), (False, True), (True, False)):
        plan.matvec_ptr(qd.data_ptr(), ph.data_ptr(), 1, False, near=near, far=far)
        r = mvp_serial(tree, ops, q, near=near, far=far) if (near, far) != (True, True) else ref
        print(env, "near" if near else "", "far" if far else "", f"{rel_l2(ph.cpu().numpy(), r):.2e}", flush=True)
    plan.close()
