"""C5 (N = 200k, 64 plane waves, P = 64, Q = 48): ms per 64-RHS product with
the right-hand-side blocks spread over 1..16 plans / streams (RhsLanes).

    python tools/lanes_sweep.py
"""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1801_03589_b200 as nesa
from paper_1801_03589_b200.plan import NesaPlan
from paper_1801_03589_b200.fastmvp import RhsLanes
n = 200_000
spec = nesa.CurveSpec(kind="ellipse-plates", seed=4)
pts = nesa.generate_sources(spec, n)
q = nesa.plane_wave_rhs(pts, nesa.wavenumber(spec, n), 64).astype(np.complex64)
qd = torch.from_numpy(np.ascontiguousarray(q)).cuda(); phi = torch.empty_like(qd)
st = torch.cuda.current_stream()
tree = nesa.build_tree(pts, nesa.TreeParams(P=64))
plan = NesaPlan(tree, nesa.build_tables(tree, nesa.NesaParams(Q=48)), dtype="f32")
for L in (1, 2, 4, 6, 8, 16):
    eng = RhsLanes(plan, L) if L > 1 else plan
    for _ in range(3): eng.matvec_ptr(qd.data_ptr(), phi.data_ptr(), 64, True, stream=st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5): eng.matvec_ptr(qd.data_ptr(), phi.data_ptr(), 64, True, stream=st.cuda_stream)
    e1.record(st); e1.synchronize()
    print(L, round(e0.elapsed_time(e1) / 5, 3), 'ms', flush=True)
    if L > 1:
        for p in eng.plans[1:]: p.close()
