"""GPU benchmark harness (run_benchmark, the gpu / gpu_dense / verify modes)
and the exact O(N^2) sum on the GPU (dense.py:14-33), SURVEY.md §8f row 4.

CPU tests: BenchConfig validation (bench.py:21-50 contract) and the Chrome
trace schema (metrics.py:67-79).  GPU tests: dense_matvec_gpu against the
oracle's restatement of dense_matvec, the reference's accuracy test
(test_fastmvp.py:50-54: full product vs dense <= 1e-4) on the GPU, and the
NESA product against the exact sum at N = 200k, where the CPU dense loop
would take ~16 minutes.
"""

import json
import os

import numpy as np
import pytest

from oracle.mvp_oracle import dense_matvec as oracle_dense, rel_l2
from paper_1801_03589_b200 import geometry as geo
from paper_1801_03589_b200.benchmark import (CSV_HEADER, BenchConfig, run_benchmark,
                                             timeline_to_chrome)


@pytest.mark.parametrize("kw", [{"n": 1}, {"repeats": 0}, {"modes": ("serial",)},
                                {"part": "both"}, {"dtype": "f16"}, {"matvecs_per_sample": 0}])
def test_config_validation(kw):
    with pytest.raises(ValueError):
        BenchConfig(**kw)


def test_chrome_trace_schema_and_lanes():
    spans = [{"name": "a", "grid": 4, "start_us": 0.0, "end_us": 10.0},
             {"name": "b", "grid": 8, "start_us": 5.0, "end_us": 20.0},
             {"name": "c", "grid": 2, "start_us": 12.0, "end_us": 15.0}]
    ev = timeline_to_chrome(spans)
    assert [e["tid"] for e in ev] == [0, 1, 0]
    for e in ev:
        assert e["ph"] == "X" and e["pid"] == 1 and e["dur"] >= 0
        assert set(e) >= {"name", "ph", "ts", "dur", "pid", "tid"}


def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.fail("GPU test without a CUDA device")
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("cplx", [False, True])
def test_dense_gpu_matches_oracle(cplx):
    _cuda()
    from paper_1801_03589_b200 import dense_matvec_gpu
    pts = geo.generate_sources(geo.CurveSpec(), 1500)
    rng = np.random.default_rng(0)
    q = rng.standard_normal(1500) + (1j * rng.standard_normal(1500) if cplx else 0)
    ref = oracle_dense(pts, q.real) + (1j * oracle_dense(pts, q.imag) if cplx else 0)
    assert rel_l2(dense_matvec_gpu(pts, q), ref) <= 1e-12


@pytest.mark.gpu
def test_dense_gpu_errors():
    _cuda()
    from paper_1801_03589_b200 import dense_matvec_gpu
    pts = geo.generate_sources(geo.CurveSpec(), 64)
    with pytest.raises(ValueError):
        dense_matvec_gpu(pts, np.ones(63))
    pts[5] = pts[9]
    with pytest.raises(ValueError, match="coincident"):
        dense_matvec_gpu(pts, np.ones(64))


@pytest.mark.gpu
def test_full_product_accuracy_vs_gpu_dense():
    # test_fastmvp.py:27-54: N = 1500 wave, P = 40, Q = 12, full vs dense <= 1e-4
    _cuda()
    from paper_1801_03589_b200 import dense_matvec_gpu, mvp
    from paper_1801_03589_b200.operators import NesaParams, build_all
    from paper_1801_03589_b200.quadtree import TreeParams, build_tree
    pts = geo.generate_sources(geo.CurveSpec(), 1500)
    tree = build_tree(pts, TreeParams(P=40))
    ops = build_all(tree, NesaParams(Q=12))
    q = np.random.default_rng(0).standard_normal(1500)
    assert rel_l2(mvp(tree, ops, q), dense_matvec_gpu(pts, q)) <= 1e-4


@pytest.mark.gpu
def test_run_benchmark_gpu_modes(tmp_path):
    _cuda()
    cfg = BenchConfig(n=20000, p_avg=50, q_aux=16, modes=("gpu", "gpu_dense", "verify"), repeats=2,
                      dtype="f64", complex_rhs=False, matvecs_per_sample=5,
                      report_out=str(tmp_path / "r.json"), trace_out=str(tmp_path / "t.json"),
                      csv_out=str(tmp_path / "c.csv"))
    rep = run_benchmark(cfg)
    assert rep["gpu"]["T_ms"] == min(rep["gpu"]["samples_ms"]) > 0
    assert rep["gpu"]["matvecs_per_s"] > 0 and rep["gpu"]["GB_s"] > 0
    assert rep["accuracy_rel_l2"] <= 1e-4        # test_acceptance.py:36-58 at Q >= 14
    assert rep["task_counts"] and rep["tree_stats"]
    assert json.load(open(tmp_path / "r.json"))["config"]["n"] == 20000
    trace = json.load(open(tmp_path / "t.json"))
    assert trace and all(e["ph"] == "X" for e in trace)
    assert any("near" in e["name"] for e in trace)
    lines = open(tmp_path / "c.csv").read().split()
    assert lines[0] == CSV_HEADER and len(lines) == 3


@pytest.mark.gpu
def test_nesa_vs_exact_sum_200k():
    # C3-sized ellipse + plates (P = 48, Q = 48), complex64 product vs the exact
    # float64 sum -- infeasible for the CPU dense loop at this size
    _cuda()
    rep = run_benchmark(BenchConfig(n=200_000, p_avg=48, q_aux=48, seed=2,
                                    curve=geo.CurveSpec(kind="ellipse-plates", seed=2),
                                    modes=("gpu", "verify"), repeats=1, matvecs_per_sample=3))
    assert rep["accuracy_rel_l2"] <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,cdt", [("f64", np.float64), ("f32", np.float32)])
def test_reference_accuracy_suite_on_gpu(dtype, cdt):
    # test_fastmvp.py:35-54 with the product and the exact sum on the GPU:
    # near exact, far == dense - near (<= 5e-4), full vs dense (<= 1e-4)
    _cuda()
    from oracle.mvp_oracle import near_mask_dense
    from paper_1801_03589_b200 import dense_matvec_gpu, mvp
    from paper_1801_03589_b200.operators import NesaParams, build_all
    from paper_1801_03589_b200.quadtree import TreeParams, build_tree
    pts = geo.generate_sources(geo.CurveSpec(), 1500)
    tree = build_tree(pts, TreeParams(P=40))
    ops = build_all(tree, NesaParams(Q=12))
    q = np.random.default_rng(0).standard_normal(1500)
    qq = q.astype(cdt)
    near = mvp(tree, ops, qq, far=False)
    far = mvp(tree, ops, qq, near=False)
    full = mvp(tree, ops, qq)
    exact = dense_matvec_gpu(pts, q)
    near_ref = near_mask_dense(tree, pts) @ q
    tol_near = 1e-13 if dtype == "f64" else 1e-6
    assert rel_l2(near, near_ref) <= tol_near
    assert rel_l2(far, exact - near_ref) <= 5e-4
    assert rel_l2(full, exact) <= 1e-4
