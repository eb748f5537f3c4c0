"""Which float32 tensor-core kernel breaks real (one-column) products? (bisect by knobs)"""
import os, subprocess, sys
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1801_03589_b200 as nesa
from paper_1801_03589_b200.plan import NesaPlan
from oracle.mvp_oracle import mvp_serial, rel_l2
n = 60000
pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=3), n)
tree = nesa.build_tree(pts, nesa.TreeParams(P=64))
params = nesa.NesaParams(Q=64)
ops = nesa.build_all(tree, params)
q = nesa.random_rhs(n, 3, complex_=False)
ref = mvp_serial(tree, ops, q, near=False)
plan = NesaPlan(tree, params, dtype="f32")
qd = torch.from_numpy(q.astype(np.float32)).cuda(); ph = torch.empty_like(qd)
plan.matvec_ptr(qd.data_ptr(), ph.data_ptr(), 1, False, near=False)
print(f"{rel_l2(ph.cpu().numpy(), ref):.2e}")
'''
for env in ({}, {"NESA_V_STORED": "1"}, {"NESA_U_STORED": "1"}, {"NESA_WIDE_LEVEL": "100000000"},
            {"NESA_V_STORED": "1", "NESA_U_STORED": "1"}, {"NESA_TC": "0"}, {"NESA_WIDE_LEVEL": "64"}):
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", CHILD, HERE], env=e, capture_output=True, text=True)
    print(env, out.stdout.strip(), out.stderr.strip()[-200:], flush=True)
