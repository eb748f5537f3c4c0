import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_1801_03589_b200 as nesa
from paper_1801_03589_b200.plan import NesaPlan
N = 2000000
pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=3), N)
tree = nesa.build_tree(pts, nesa.TreeParams(P=64))
tab = nesa.build_tables(tree, nesa.NesaParams(Q=64))
p32 = NesaPlan(tree, tab, dtype="f32")
p64 = NesaPlan(tree, tab, dtype="f64")
st = torch.cuda.current_stream()
for seed in (3, 11, 12345):
    q = nesa.random_rhs(N, seed)
    q64 = torch.from_numpy(q.astype(np.complex128)).cuda(); y64 = torch.empty_like(q64)
    q32 = torch.from_numpy(q.astype(np.complex64)).cuda(); y32 = torch.empty_like(q32)
    p64.matvec_ptr(q64.data_ptr(), y64.data_ptr(), 1, True, stream=st.cuda_stream)
    p32.matvec_ptr(q32.data_ptr(), y32.data_ptr(), 1, True, stream=st.cuda_stream)
    torch.cuda.synchronize()
    d = (y32.to(torch.complex128) - y64)
    print(seed, float(torch.linalg.norm(d) / torch.linalg.norm(y64)))
