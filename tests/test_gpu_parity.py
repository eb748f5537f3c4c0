"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden outputs and the oracle.

Tolerances (BASELINE.json north_star): relative L2 <= 1e-12 for float64 /
complex128 plans, <= 1e-5 for float32 / complex64 plans, near field alone
<= 1e-13 (test_fastmvp.py:35-40 bar) in float64.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN_CASES, grid_points
from oracle.mvp_oracle import mvp_serial as oracle_mvp, rel_l2
from paper_1801_03589_b200 import geometry as geo
from paper_1801_03589_b200 import mvp, task_counts
from paper_1801_03589_b200.operators import NesaParams, build_all
from paper_1801_03589_b200.plan import NesaPlan
from paper_1801_03589_b200.quadtree import TreeParams, build_tree

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _problem(g):
    tree = build_tree(g["points"], TreeParams(P=int(g["P"])))
    params = NesaParams(Q=int(g["Q"]))
    return tree, params


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_f64_device_assembled_vs_golden(golden, name):
    g = golden(name)
    tree, params = _problem(g)
    q = g["q"]
    assert rel_l2(mvp(tree, params, q), g["phi"]) <= 1e-12
    assert rel_l2(mvp(tree, params, q, far=False), g["phi_near"]) <= 1e-13
    assert rel_l2(mvp(tree, params, q, near=False), g["phi_far"]) <= 1e-12


@pytest.mark.parametrize("name", ["fastmvp_1500", "grid4_single_level", "c1_wave_2000",
                                  "c1_circle_2000", "annulus_1024"])
def test_f64_host_operators_vs_golden(golden, name):
    # drop-in route: host OperatorSet (build_all) uploaded as is
    g = golden(name)
    tree, params = _problem(g)
    ops = build_all(tree, params)
    q = g["q"]
    assert rel_l2(mvp(tree, ops, q), g["phi"]) <= 1e-12
    assert rel_l2(mvp(tree, ops, q, far=False), g["phi_near"]) <= 1e-13
    assert rel_l2(mvp(tree, ops, q, near=False), g["phi_far"]) <= 1e-12


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_c64_vs_golden(golden, name):
    g = golden(name)
    tree, params = _problem(g)
    q = g["q"]
    q32 = q.astype(np.complex64 if np.iscomplexobj(q) else np.float32)
    phi = mvp(tree, params, q32)
    assert phi.dtype == q32.dtype
    assert rel_l2(phi, g["phi"]) <= 1e-5


def test_zero_in_zero_out_and_wrong_length(golden):
    g = golden("fastmvp_1500")
    tree, params = _problem(g)
    z = mvp(tree, params, np.zeros(tree.n_points))
    assert (z == 0).all()
    with pytest.raises(ValueError):
        mvp(tree, params, np.ones(3))
    with pytest.raises(ValueError):
        mvp(tree, params, np.ones((tree.n_points, 2, 2)))


def test_deterministic_and_no_stale_sums(golden):
    g = golden("c1_wave_2000")
    tree, params = _problem(g)
    q = g["q"]
    a = mvp(tree, params, q)
    b = mvp(tree, params, 3.0 * q)
    c = mvp(tree, params, q)
    assert np.array_equal(a, c)                 # bitwise run-to-run
    assert rel_l2(b, 3.0 * a) <= 1e-14          # linearity, no stale sums


def test_multi_rhs_matches_columns(golden):
    g = golden("c1_circle_2000")
    tree, params = _problem(g)
    pts = g["points"]
    Qm = geo.plane_wave_rhs(tree.points[np.argsort(tree.perm)], 4.0, n_waves=2)
    ref = np.stack([g["phi"]], 1)
    phi = mvp(tree, params, Qm)
    assert phi.shape == Qm.shape
    ops = build_all(tree, params)
    exp = oracle_mvp(tree, ops, Qm)
    assert rel_l2(phi, exp) <= 1e-12
    del ref, pts


def test_single_level_tree():
    pts = grid_points(4)
    tree = build_tree(pts, TreeParams(P=16))
    params = NesaParams(Q=14)
    q = np.random.default_rng(1).standard_normal(16)
    counts = task_counts(tree)
    assert counts["source-transfer"] == 0
    assert rel_l2(mvp(tree, params, q), oracle_mvp(tree, build_all(tree, params), q)) <= 1e-12


def test_permutation_equivariance():
    # test_fastmvp.py:156-168
    pts = geo.generate_sources(geo.CurveSpec(), 1500)
    rng = np.random.default_rng(5)
    perm = rng.permutation(len(pts))
    q = rng.standard_normal(len(pts))
    ta = build_tree(pts, TreeParams(P=40))
    tb = build_tree(pts[perm], TreeParams(P=40))
    p = NesaParams(Q=12)
    phi_a = mvp(ta, p, q)
    phi_b = mvp(tb, p, q[perm])
    np.testing.assert_allclose(phi_b, phi_a[perm], rtol=1e-10, atol=1e-12)


def test_torch_device_tensors_roundtrip(golden):
    g = golden("c1_wave_2000")
    tree, params = _problem(g)
    qd = torch.from_numpy(g["q"]).cuda()
    phi = mvp(tree, params, qd)
    assert phi.is_cuda and phi.dtype == torch.complex128
    assert rel_l2(phi.cpu().numpy(), g["phi"]) <= 1e-12


def test_large_tall_leaves_paneled():
    # leaves with > 512 points exercise the row panels of near and U
    pts = geo.generate_sources(geo.CurveSpec(), 6000)
    tree = build_tree(pts, TreeParams(P=700))
    assert max(g.n_points for g in tree.leaves()) > 512
    params = NesaParams(Q=12)
    q = np.random.default_rng(3).standard_normal(6000)
    ops = build_all(tree, params)
    assert rel_l2(mvp(tree, params, q), oracle_mvp(tree, ops, q)) <= 1e-12


def test_plan_stats(golden):
    g = golden("c2_wave_20000")
    tree, params = _problem(g)
    plan = NesaPlan(tree, params, dtype="f32")
    a = tree.arrays
    sizes = a.stop - a.start
    e_near = sum(int(sizes[i]) * int(sizes[a.nbr_idx[a.nbr_ptr[i]:a.nbr_ptr[i + 1]]].sum())
                 for i in range(a.level_count[tree.L]))
    assert plan.stat("near_entries") == e_near
    # float32 plans from geometry: radiation and reception through circle
    # expansions, no stored V / U
    assert plan.stat("v_entries") == 0 and plan.stat("u_entries") == 0
    assert 8 <= plan.stat("v_moments") <= 96 and 4 <= plan.stat("u_terms") <= 96
    assert plan.stat("d_refs") == int(a.int_ptr[-1])
    plan.close()
    # float64 plans: stored V (the pinv fit on the host), reception through
    # the incoming expansion in float64 (more terms than float32)
    plan = NesaPlan(tree, params, dtype="f64")
    assert plan.stat("v_entries") == tree.n_points * params.Q
    assert plan.stat("u_entries") == 0 and plan.stat("v_moments") == 0
    assert plan.stat("u_terms") > 4 and plan.stat("u_terms") <= 96
    plan.close()


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_q64_bench_geometry_vs_oracle(dtype, tol):
    # the benchmark's configuration family (ellipse + plates, P=64, Q=64) at a
    # size the oracle finishes in seconds; exercises the Q=64 fast paths
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=3), 30000)
    tree = build_tree(pts, TreeParams(P=64))
    params = NesaParams(Q=64)
    q = geo.random_rhs(30000, 3)
    ref = oracle_mvp(tree, build_all(tree, params), q)
    qq = q if dtype == "f64" else q.astype(np.complex64)
    assert rel_l2(mvp(tree, params, qq), ref) <= tol


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_q64_wide_level_kernels(monkeypatch, dtype, tol):
    # force the warp-tiled level kernels onto a tree the oracle can check
    monkeypatch.setenv("NESA_WIDE_LEVEL", "32")
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=5), 40000)
    tree = build_tree(pts, TreeParams(P=64))
    params = NesaParams(Q=64)
    plan = NesaPlan(tree, params, dtype=dtype)
    q = geo.random_rhs(40000, 5)
    qq = q if dtype == "f64" else q.astype(np.complex64)
    qd = torch.from_numpy(qq).cuda()
    phi = torch.empty_like(qd)
    plan.matvec_ptr(qd.data_ptr(), phi.data_ptr(), 1, True,
                    stream=torch.cuda.current_stream().cuda_stream)
    ref = oracle_mvp(tree, build_all(tree, params), q)
    assert rel_l2(phi.cpu().numpy(), ref) <= tol
    plan.close()


@pytest.mark.parametrize("world,dtype,tol", [(2, "f64", 1e-12), (3, "f32", 1e-5)])
def test_subplans_with_exchange_on_one_gpu(world, dtype, tol):
    # the multi-GPU path's kernels: per-rank sub-plans (leaf ranges, partial
    # upward sums, stage 1 / stage 2 graphs) run one after another on one
    # device; the all_gather is a concatenation of the ranks' send buffers
    from paper_1801_03589_b200.dist import (build_exchange, combine_s, exchange_tensors, pack_s,
                                            partition_leaves)
    from paper_1801_03589_b200.dist import _tensor_from_ptr
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=2), 20000)
    tree = build_tree(pts, TreeParams(P=32))
    params = NesaParams(Q=24)
    ranges = partition_leaves(tree, world, params.Q)
    q = geo.random_rhs(20000, 2)
    cdt = np.complex128 if dtype == "f64" else np.complex64
    qd = torch.from_numpy(q.astype(cdt)).cuda()
    st = torch.cuda.current_stream().cuda_stream
    plans, phis, xps, tens, svs = [], [], [], [], []
    G = tree.arrays.n_groups
    tdt = torch.float64 if dtype == "f64" else torch.float32
    for r in range(world):
        p = NesaPlan(tree, params, dtype=dtype, leaf_range=ranges[r])
        phi = torch.zeros_like(qd)
        p.matvec_ptr(qd.data_ptr(), phi.data_ptr(), 1, True, stream=st, stage=1)
        sv = _tensor_from_ptr(p.s_dev_ptr(2), (G, params.Q * 2), tdt, 0)
        xp = build_exchange(tree, ranges, r)
        plans.append(p), phis.append(phi), xps.append(xp), svs.append(sv)
        tens.append(exchange_tensors(xp, sv.device))
    sends = [pack_s(svs[r], xps[r], tens[r]) for r in range(world)]
    recv = torch.cat(sends, 0)
    for r in range(world):
        combine_s(svs[r], xps[r], recv, tens[r])
    total = torch.zeros_like(qd)
    for r in range(world):
        plans[r].matvec_ptr(qd.data_ptr(), phis[r].data_ptr(), 1, True, stream=st, stage=2)
        total += phis[r]
    ref = oracle_mvp(tree, build_all(tree, params), q)
    assert rel_l2(total.cpu().numpy(), ref) <= tol
    for p in plans:
        p.close()


def test_pinned_host_tensor_roundtrip(golden):
    g = golden("c1_circle_2000")
    tree, params = _problem(g)
    qh = torch.from_numpy(g["q"].astype(np.complex64)).pin_memory()
    phi = mvp(tree, params, qh)
    assert not phi.is_cuda and phi.is_pinned() and phi.dtype == torch.complex64
    assert rel_l2(phi.numpy(), g["phi"]) <= 1e-5


@pytest.mark.parametrize("dtype,tol,nrhs,cplx", [("f64", 1e-12, 7, True), ("f32", 1e-5, 5, False),
                                                 ("f32", 1e-5, 16, True)])
def test_many_rhs_column_blocks(dtype, tol, nrhs, cplx):
    # C5: many right-hand sides (plane waves) run as column blocks of <= 4 reals
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=4), 8000)
    tree = build_tree(pts, TreeParams(P=32))
    params = NesaParams(Q=24)
    k = geo.wavenumber(geo.CurveSpec(kind="ellipse-plates", seed=4), 8000)
    Qm = geo.plane_wave_rhs(pts, k, n_waves=nrhs)
    if not cplx:
        Qm = Qm.real.copy()
    ref = oracle_mvp(tree, build_all(tree, params), Qm)
    qq = Qm if dtype == "f64" else Qm.astype(np.complex64 if cplx else np.float32)
    phi = mvp(tree, params, qq)
    assert phi.shape == Qm.shape
    assert rel_l2(phi, ref) <= tol


@pytest.mark.parametrize("name", ["fastmvp_1500", "c1_wave_2000", "c2_circle_20000",
                                  "ellipse_plates_20000"])
def test_f32_near_and_far_parts(golden, name):
    # float32 plans compute the near field and the reception matrix-free
    g = golden(name)
    tree, params = _problem(g)
    q = g["q"].astype(np.complex64 if np.iscomplexobj(g["q"]) else np.float32)
    assert rel_l2(mvp(tree, params, q, far=False), g["phi_near"]) <= 1e-5
    assert rel_l2(mvp(tree, params, q, near=False), g["phi_far"]) <= 1e-5


def test_f32_tall_leaves_matrix_free():
    pts = geo.generate_sources(geo.CurveSpec(), 6000)
    tree = build_tree(pts, TreeParams(P=700))
    assert max(g.n_points for g in tree.leaves()) > 160
    params = NesaParams(Q=12)
    q = np.random.default_rng(3).standard_normal(6000)
    ref = oracle_mvp(tree, build_all(tree, params), q)
    assert rel_l2(mvp(tree, params, q.astype(np.float32)), ref) <= 1e-5


@pytest.mark.parametrize("name", ["c1_wave_2000", "c2_circle_20000", "ellipse_plates_20000"])
def test_f32_stored_v_u_paths(monkeypatch, golden, name):
    # the stored-operator float32 paths (blockgemv V / U) stay correct when the
    # circle expansions are switched off
    monkeypatch.setenv("NESA_V_STORED", "1")
    monkeypatch.setenv("NESA_U_STORED", "1")
    g = golden(name)
    tree, params = _problem(g)
    q = g["q"].astype(np.complex64 if np.iscomplexobj(g["q"]) else np.float32)
    plan = NesaPlan(tree, params, dtype="f32")
    assert plan.stat("v_moments") == 0 and plan.stat("u_terms") == 0
    assert plan.stat("v_entries") == tree.n_points * params.Q
    plan.close()
    assert rel_l2(mvp(tree, params, q), g["phi"]) <= 1e-5


@pytest.mark.parametrize("nm,nt", [(8, 4), (96, 96)])
def test_f32_expansion_term_counts(monkeypatch, golden, nm, nt):
    # forced term counts: too few terms must show up as error, many terms
    # must stay within the float32 tolerance (no overflow / breakdown)
    monkeypatch.setenv("NESA_V_MOMENTS", str(nm))
    monkeypatch.setenv("NESA_U_TERMS", str(nt))
    g = golden("ellipse_plates_20000")
    tree, params = _problem(g)
    q = g["q"].astype(np.complex64 if np.iscomplexobj(g["q"]) else np.float32)
    err = rel_l2(mvp(tree, params, q, near=False), g["phi_far"])
    if nm >= 64:
        assert err <= 1e-5
    else:
        assert err > 1e-5


def test_pipeline_matches_sync_calls(golden):
    # overlapped host-to-host products give exactly the synchronous results
    import torch
    from paper_1801_03589_b200 import MvpPipeline
    g = golden("ellipse_plates_20000")
    tree, params = _problem(g)
    rng = np.random.default_rng(5)
    n = tree.n_points
    qs = [torch.from_numpy((rng.standard_normal(n) + 1j * rng.standard_normal(n))
                           .astype(np.complex64)).pin_memory() for _ in range(5)]
    outs = [torch.empty_like(q).pin_memory() for q in qs]
    pipe = MvpPipeline(tree, params, dtype="f32", is_complex=True)
    for q, o in zip(qs, outs):
        pipe.submit(q, o)
    pipe.synchronize()
    for q, o in zip(qs, outs):
        ref = mvp(tree, params, q.numpy())
        assert np.array_equal(o.numpy(), ref)
    with pytest.raises(ValueError):
        pipe.submit(qs[0][:-1], outs[0])


@pytest.mark.parametrize("env", [{}, {"NESA_TC": "0"}])
def test_q64_f32_path_variants(monkeypatch, env):
    # the float32 Q = 64 translation on the tensor cores (default) and with
    # the FFMA kernel float64 plans use, against the oracle
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=7), 30000)
    tree = build_tree(pts, TreeParams(P=64))
    params = NesaParams(Q=64)
    q = geo.random_rhs(30000, 7)
    ref = oracle_mvp(tree, build_all(tree, params), q)
    plan = NesaPlan(tree, params, dtype="f32")
    qd = torch.from_numpy(q.astype(np.complex64)).cuda()
    phi = torch.empty_like(qd)
    plan.matvec_ptr(qd.data_ptr(), phi.data_ptr(), 1, True,
                    stream=torch.cuda.current_stream().cuda_stream)
    assert rel_l2(phi.cpu().numpy(), ref) <= 1e-5
    plan.close()


def test_tensor_core_translation_kernel_standalone(tmp_path):
    # tools/tc_test.cu: the tcgen05 tf32x3 GEMM against a float64 host
    # reference for R = 1, 2, 4 (single- and multi-tile units)
    import shutil
    import subprocess
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "tc_test")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
                    "-o", exe, os.path.join(root, "tools", "tc_test.cu")], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "PASS" in out.stdout, out.stdout


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-9), ("f32", 2e-5)])
def test_gmres_solves_shifted_system(dtype, tol):
    # (shift I + K~) x = b with 3 right-hand sides solved side by side; the
    # residual is re-checked with the CPU oracle product
    from paper_1801_03589_b200 import gmres
    pts = geo.generate_sources(geo.CurveSpec(), 3000)
    tree = build_tree(pts, TreeParams(P=32))
    params = NesaParams(Q=24)
    ops = build_all(tree, params)
    rng = np.random.default_rng(11)
    b = rng.standard_normal((3000, 3)) + 1j * rng.standard_normal((3000, 3))
    shift = 50.0
    bb = b if dtype == "f64" else b.astype(np.complex64)
    res = gmres(tree, params, bb, shift=shift, tol=tol, restart=30, maxiter=300)
    assert res.converged.all(), res.residuals
    x = np.asarray(res.x, dtype=np.complex128)
    r = b - (shift * x + oracle_mvp(tree, ops, x))
    rel = np.linalg.norm(r, axis=0) / np.linalg.norm(b, axis=0)
    assert (rel <= 5 * tol).all(), rel
    # single column, torch CUDA input -> CUDA output
    bt = torch.from_numpy(bb[:, 0].copy()).cuda()
    r1 = gmres(tree, params, bt, shift=shift, tol=tol, restart=30, maxiter=300)
    assert r1.x.is_cuda and r1.converged.all()
    assert np.allclose(r1.x.cpu().numpy(), np.asarray(res.x)[:, 0], rtol=0, atol=20 * tol * np.abs(x).max())


def test_loaded_problem_gives_identical_products(tmp_path):
    from paper_1801_03589_b200 import load_problem, save_problem
    from paper_1801_03589_b200.operators import build_tables
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=9), 30000)
    tree = build_tree(pts, TreeParams(P=64))
    tables = build_tables(tree, NesaParams(Q=64))
    save_problem(str(tmp_path / "p.npz"), tree, tables)
    t2, tab2 = load_problem(str(tmp_path / "p.npz"))
    q = geo.random_rhs(30000, 9).astype(np.complex64)
    assert np.array_equal(mvp(tree, tables, q), mvp(t2, tab2, q))


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_q48_split_and_fused_levels(monkeypatch, dtype, tol):
    # Q != 64 with several "wide" levels: the side-stream translation split
    # must sit outside the fused coarse range (regression: C3 capture error)
    monkeypatch.setenv("NESA_WIDE_LEVEL", "64")
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=2), 30000)
    tree = build_tree(pts, TreeParams(P=48))
    params = NesaParams(Q=48)
    q = geo.random_rhs(30000, 2)
    ref = oracle_mvp(tree, build_all(tree, params), q)
    qq = q if dtype == "f64" else q.astype(np.complex64)
    assert rel_l2(mvp(tree, params, qq), ref) <= tol


@pytest.mark.parametrize("dtype,cdt", [("f32", np.complex64), ("f64", np.complex128)])
def test_rhs_lanes_bitwise_and_vs_oracle(dtype, cdt):
    # many right-hand sides spread over 3 plans on 3 streams: every bit equals
    # the single-plan multi-column product, and each column the oracle
    from paper_1801_03589_b200.fastmvp import RhsLanes
    pts = geo.generate_sources(geo.CurveSpec(kind="circle-random", seed=1), 20000)
    tree = build_tree(pts, TreeParams(P=32))
    params = NesaParams(Q=32)
    rng = np.random.default_rng(5)
    q = (rng.standard_normal((20000, 11)) + 1j * rng.standard_normal((20000, 11))).astype(cdt)
    plan = NesaPlan(tree, params, dtype=dtype)
    lanes = RhsLanes(plan, 3)
    qd = torch.from_numpy(q).cuda()
    a, b = torch.empty_like(qd), torch.empty_like(qd)
    st = torch.cuda.current_stream().cuda_stream
    plan.matvec_ptr(qd.data_ptr(), a.data_ptr(), 11, True, stream=st)
    lanes.matvec_ptr(qd.data_ptr(), b.data_ptr(), 11, True, stream=st)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    ops = build_all(tree, params)
    tol = 1e-12 if dtype == "f64" else 1e-5
    for j in (0, 5, 10):
        assert rel_l2(b[:, j].cpu().numpy(), oracle_mvp(tree, ops, q[:, j].astype(np.complex128))) <= tol
    for p in lanes.plans[1:]:
        p.close()
    plan.close()


@pytest.mark.parametrize("tdt", ["float32", "float64"])
def test_exchange_kernels_match_torch_ops(tdt):
    # nesa_exchange_pack / _combine (CUDA) bitwise against the torch-op
    # version the gloo tests run on CPU
    from paper_1801_03589_b200.dist import (build_exchange, combine_s, exchange_tensors, pack_s,
                                            partition_leaves)
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=2), 20000)
    tree = build_tree(pts, TreeParams(P=32))
    world = 4
    ranges = partition_leaves(tree, world, 24)
    G = tree.arrays.n_groups
    dt = getattr(torch, tdt)
    gen = torch.Generator().manual_seed(3)
    s_cpu = [torch.randn((G, 48), generator=gen, dtype=dt) for _ in range(world)]
    xps = [build_exchange(tree, ranges, r) for r in range(world)]
    outs = {}
    for dev in ("cpu", "cuda"):
        ss = [x.clone().to(dev) for x in s_cpu]
        tens = [exchange_tensors(xp, ss[0].device) for xp in xps]
        sends = [pack_s(ss[r], xps[r], tens[r]) for r in range(world)]
        recv = torch.cat(sends, 0)
        for r in range(world):
            combine_s(ss[r], xps[r], recv, tens[r])
        outs[dev] = ([x.cpu() for x in sends], [x.cpu() for x in ss])
    for a, b in zip(outs["cpu"][0], outs["cuda"][0]):
        assert torch.equal(a, b)
    for a, b in zip(outs["cpu"][1], outs["cuda"][1]):
        assert torch.equal(a, b)


def test_graph_cache_repoints_buffers_without_recapture():
    # one captured graph per (width, flags, stage); new q / phi buffers are
    # patched into the instantiated graph, so 50 distinct buffer pairs do not
    # grow the cache and every product is exact (bitwise equal to the first)
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=6), 6000)
    tree = build_tree(pts, TreeParams(P=32))
    params = NesaParams(Q=24)
    plan = NesaPlan(tree, params, dtype="f32")
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(8)
    qs = [torch.from_numpy((rng.standard_normal(6000) + 1j * rng.standard_normal(6000))
                           .astype(np.complex64)).cuda() for _ in range(5)]
    first = {}
    keep = []
    for it in range(50):
        k = it % 5
        q = qs[k].clone()          # a fresh buffer every time
        phi = torch.empty_like(q)
        keep.append((q, phi))      # keep them alive: every pointer stays distinct
        plan.matvec_ptr(q.data_ptr(), phi.data_ptr(), 1, True, stream=st)
        if k in first:
            assert torch.equal(phi, first[k])
        else:
            first[k] = phi.clone()
    torch.cuda.synchronize()
    assert plan.stat("graph_captures") == 1
    assert plan.stat("graphs_cached") == 1
    ops = build_all(tree, params)
    for k in (0, 3):
        ref = oracle_mvp(tree, ops, qs[k].cpu().numpy().astype(np.complex128))
        assert rel_l2(first[k].cpu().numpy(), ref) <= 1e-5
    plan.close()


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_mixed_widths_on_one_plan(dtype, tol):
    # regression (round-1 advisor): real -> complex -> 2 complex -> real on ONE
    # plan with buffers the caching allocator hands back; growing the
    # workspace must not leave a graph addressing freed memory
    pts = geo.generate_sources(geo.CurveSpec(kind="circle-random", seed=3), 8000)
    tree = build_tree(pts, TreeParams(P=32))
    params = NesaParams(Q=20)
    ops = build_all(tree, params)
    plan = NesaPlan(tree, params, dtype=dtype)
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(4)
    rdt = torch.float64 if dtype == "f64" else torch.float32
    cdt = torch.complex128 if dtype == "f64" else torch.complex64
    cases = [(rng.standard_normal(8000), False, 1),
             (rng.standard_normal(8000) + 1j * rng.standard_normal(8000), True, 1),
             (rng.standard_normal((8000, 2)) + 1j * rng.standard_normal((8000, 2)), True, 2),
             (rng.standard_normal(8000), False, 1)]
    for q, cplx, nrhs in cases:
        qd = torch.from_numpy(q).to("cuda", dtype=cdt if cplx else rdt)
        phi = torch.empty_like(qd)
        plan.matvec_ptr(qd.data_ptr(), phi.data_ptr(), nrhs, cplx, stream=st)
        ref = oracle_mvp(tree, ops, q)
        assert rel_l2(phi.cpu().numpy(), ref) <= tol
        del qd, phi
    plan.close()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_distributed_plan_one_rank_matches_plan(dtype):
    # the in-graph exchange path (nesa_plan_create_dist: pack -> ncclAllGather
    # -> combine captured into the product graph) on a one-rank NCCL
    # communicator: bitwise the single-plan product (multi-rank correctness
    # of the exchange tables is covered by the gloo tests)
    import torch.distributed as dist
    from paper_1801_03589_b200.dist import DistNesa
    if not dist.is_initialized():
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=3), 40000)
    tree = build_tree(pts, TreeParams(P=64))
    params = NesaParams(Q=64)
    eng = DistNesa(tree, params, dtype=dtype, device=0)
    plan = NesaPlan(tree, params, dtype=dtype)
    cdt = np.complex64 if dtype == "f32" else np.complex128
    q = torch.from_numpy(geo.random_rhs(40000, 3).astype(cdt)).cuda()
    a, b = torch.zeros_like(q), torch.zeros_like(q)
    st = torch.cuda.current_stream().cuda_stream
    eng.matvec_ptr(q.data_ptr(), a.data_ptr(), 1, True, stream=st)
    plan.matvec_ptr(q.data_ptr(), b.data_ptr(), 1, True, stream=st)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    eng.close()
    plan.close()


@pytest.mark.parametrize("Q,P", [(48, 64), (64, 64), (24, 32)])
def test_c5_plane_waves_near_on_tensor_cores(Q, P):
    # C5 (BASELINE configs[4]) at a reduced size: 64 plane waves = 128 real
    # columns.  float32 plans run the near field as ONE tcgen05 GEMM over all
    # columns (nesa_matvec_near_wide) and the far field in 4-column blocks;
    # every column against the oracle, and the lanes path (extra far-only
    # plans) bitwise equal to the one-plan product
    from paper_1801_03589_b200.fastmvp import RhsLanes
    n = 20000
    spec = geo.CurveSpec(kind="ellipse-plates", seed=4)
    pts = geo.generate_sources(spec, n)
    tree = build_tree(pts, TreeParams(P=P))
    params = NesaParams(Q=Q)
    k = geo.wavenumber(spec, n)
    Qm = geo.plane_wave_rhs(pts, k, n_waves=64)
    plan = NesaPlan(tree, params, dtype="f32")
    assert plan.stat("near_wide") == 1
    qd = torch.from_numpy(Qm.astype(np.complex64)).cuda()
    a, b = torch.empty_like(qd), torch.empty_like(qd)
    st = torch.cuda.current_stream().cuda_stream
    plan.matvec_ptr(qd.data_ptr(), a.data_ptr(), 64, True, stream=st)
    lanes = RhsLanes(plan, 4)
    assert all(p.far_only for p in lanes.plans[1:])
    lanes.matvec_ptr(qd.data_ptr(), b.data_ptr(), 64, True, stream=st)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    ops = build_all(tree, params)
    cols = [0, 17, 63]
    ref = oracle_mvp(tree, ops, Qm[:, cols])
    got = a.cpu().numpy()[:, cols]
    for j in range(len(cols)):
        assert rel_l2(got[:, j], ref[:, j]) <= 1e-5
    # the near field alone (wide GEMM) against the oracle's near part
    c = torch.zeros_like(qd)
    plan.near_wide_ptr(qd.data_ptr(), c.data_ptr(), 128, 0, 128, stream=st)
    torch.cuda.synchronize()
    refn = oracle_mvp(tree, ops, Qm[:, cols], far=False)
    for j, col in enumerate(cols):
        assert rel_l2(c.cpu().numpy()[:, col], refn[:, j]) <= 1e-5
    for p in lanes.plans[1:]:
        p.close()
    plan.close()


@pytest.mark.parametrize("dt,kk,tol", [(torch.complex64, 7, 2e-5), (torch.complex128, 31, 1e-12),
                                       (torch.complex64, 40, 2e-5)])
def test_fused_gram_schmidt_step(dt, kk, tol):
    # nesa_gs_step (three passes, Hessenberg column on the device) against
    # CGS2 in float64 numpy: same h column, same normalised new basis vector
    from paper_1801_03589_b200 import _capi
    lib = _capi.load()
    n = 50000
    rng = np.random.default_rng(kk)
    Vh = np.linalg.qr(rng.standard_normal((n, kk)) + 1j * rng.standard_normal((n, kk)))[0].T.copy()
    wh = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    h1 = Vh.conj() @ wh
    w1 = wh - Vh.T @ h1
    h2 = Vh.conj() @ w1
    w2 = w1 - Vh.T @ h2
    nrm = np.linalg.norm(w2)
    V = torch.zeros((kk + 1, n), dtype=dt, device="cuda")
    V[:kk] = torch.from_numpy(Vh).to(V)
    w = torch.from_numpy(wh).to("cuda", dt)
    work = torch.zeros(int(lib.nesa_gs_work_bytes()), dtype=torch.uint8, device="cuda")
    hcol = torch.zeros(2 * (kk + 1), dtype=torch.float64, device="cuda")
    stride = (V[1].data_ptr() - V[0].data_ptr()) // (V.element_size() // 2)
    rc = lib.nesa_gs_step(V.data_ptr(), stride, kk, w.data_ptr(), V[kk].data_ptr(), n,
                          int(dt == torch.complex128), work.data_ptr(), hcol.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    h = hcol.cpu().numpy()
    hc = h[0:2 * kk:2] + 1j * h[1:2 * kk:2]
    assert np.abs(hc - (h1 + h2)).max() <= tol * np.abs(h1).max()
    assert abs(h[2 * kk] - nrm) <= tol * nrm
    assert np.linalg.norm(V[kk].cpu().numpy() - w2 / nrm) <= 10 * tol


@pytest.mark.parametrize("dtype,tol,nw,Q,P", [("f32", 1e-5, 70, 24, 32), ("f32", 1e-5, 64, 96, 64),
                                              ("f64", 1e-12, 9, 48, 32)])
def test_many_rhs_far_field_as_gemms(dtype, tol, nw, Q, P):
    # C5: more than 4 real columns on a plan with stored V / U run the far
    # field as batched GEMMs over 128-column passes (wgemm_kernel) -- here 140
    # real columns (two passes), Q = 96 (two row tiles per group) and the
    # float64 engine (far field only: its near field has no tensor-core path)
    from paper_1801_03589_b200.fastmvp import get_plan
    n = 12000
    spec = geo.CurveSpec(kind="ellipse-plates", seed=4)
    pts = geo.generate_sources(spec, n)
    tree = build_tree(pts, TreeParams(P=P))
    params = NesaParams(Q=Q)
    Qm = geo.plane_wave_rhs(pts, geo.wavenumber(spec, n), n_waves=nw)
    ops = build_all(tree, params)
    cols = [0, nw // 2, nw - 1]
    qq = Qm if dtype == "f64" else Qm.astype(np.complex64)
    near = dtype == "f32"
    phi = mvp(tree, params, qq, near=near)
    assert get_plan(tree, params, dtype=dtype, wide=True).stat("far_wide") == 1
    ref = oracle_mvp(tree, ops, Qm[:, cols], near=near)
    for j, c in enumerate(cols):
        assert rel_l2(phi[:, c], ref[:, j]) <= tol, (c, rel_l2(phi[:, c], ref[:, j]))


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_q128_warp_tiled_levels_and_translation(monkeypatch, dtype, tol):
    # Q = 128: the warp-tiled level kernels (forced onto every level with
    # >= 64 groups) and translation at their largest operator size
    monkeypatch.setenv("NESA_WIDE_LEVEL", "64")
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=5), 12000)
    tree = build_tree(pts, TreeParams(P=32))
    params = NesaParams(Q=128)
    q = geo.random_rhs(12000, 5)
    ref = oracle_mvp(tree, build_all(tree, params), q)
    qq = q if dtype == "f64" else q.astype(np.complex64)
    plan = NesaPlan(tree, params, dtype=dtype)
    qd = torch.from_numpy(qq).cuda()
    ph = torch.empty_like(qd)
    plan.matvec_ptr(qd.data_ptr(), ph.data_ptr(), 1, True)
    err = rel_l2(ph.cpu().numpy(), ref)
    plan.close()
    assert err <= tol, err


@pytest.mark.parametrize("n", [60000, 200000])
def test_real_charges_float32_q64(n):
    # the reference's own input: real charges (fastmvp.py:145-146), on the
    # float32 Q = 64 bench-geometry plan (moment radiation, tensor-core
    # levels / translation, expansion reception) -- one real column
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=3), n)
    tree = build_tree(pts, TreeParams(P=64))
    params = NesaParams(Q=64)
    q = geo.random_rhs(n, 3, complex_=False)
    ops = build_all(tree, params)
    for near, far in ((True, True), (False, True)):
        ref = oracle_mvp(tree, ops, q, near=near, far=far)
        phi = mvp(tree, params, q.astype(np.float32), near=near, far=far)
        assert phi.dtype == np.float32
        assert rel_l2(phi, ref) <= 1e-5, (near, far, rel_l2(phi, ref))


@pytest.mark.parametrize("dtype,tol", [("f32", 1e-5), ("f64", 1e-12)])
@pytest.mark.parametrize("cplx,nrhs", [(False, 1), (False, 2), (False, 3), (False, 4), (True, 1),
                                       (True, 2)])
def test_column_count_matrix_q64(dtype, tol, cplx, nrhs):
    # every vector width the engine specialises (R = 1, 2, 4 real columns per
    # block; complex = column pairs) on the Q = 64 bench geometry, whose float32
    # plan runs the tensor-core and expansion kernels
    n = 30000
    pts = geo.generate_sources(geo.CurveSpec(kind="ellipse-plates", seed=6), n)
    tree = build_tree(pts, TreeParams(P=64))
    params = NesaParams(Q=64)
    rng = np.random.default_rng(6)
    q = rng.standard_normal((n, nrhs)) + (1j * rng.standard_normal((n, nrhs)) if cplx else 0.0)
    if nrhs == 1:
        q = q[:, 0]
    ref = oracle_mvp(tree, build_all(tree, params), q)
    if dtype == "f32":
        q = q.astype(np.complex64 if cplx else np.float32)
    assert rel_l2(mvp(tree, params, q), ref) <= tol
