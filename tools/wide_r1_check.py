import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
os.environ["NESA_WIDE_LEVEL"] = "64"
import paper_1801_03589_b200 as nesa
from paper_1801_03589_b200.plan import NesaPlan
from oracle.mvp_oracle import mvp_serial, rel_l2
pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=5), 12000)
tree = nesa.build_tree(pts, nesa.TreeParams(P=32))
for Q in (64, 128):
    params = nesa.NesaParams(Q=Q)
    ops = nesa.build_all(tree, params)
    for cplx in (False, True):
        q = nesa.random_rhs(12000, 5, complex_=cplx)
        ref = mvp_serial(tree, ops, q)
        for dt in ("f64", "f32"):
            qq = q if dt == "f64" else q.astype(np.complex64 if cplx else np.float32)
            plan = NesaPlan(tree, params, dtype=dt)
            qd = torch.from_numpy(qq).cuda(); ph = torch.empty_like(qd)
            plan.matvec_ptr(qd.data_ptr(), ph.data_ptr(), 1, cplx)
            print(Q, "complex" if cplx else "real", dt, f"{rel_l2(ph.cpu().numpy(), ref):.2e}", flush=True)
            plan.close()
