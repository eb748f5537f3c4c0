"""Benchmark harness with a GPU mode (reference: bench.py:21-188).

Mirrors the reference's ``BenchConfig`` / ``run_benchmark(config)`` report
contract for the modes that exist here:

* ``gpu``       -- the NESA product on the B200 (``NesaPlan`` CUDA graph):
                   samples / T_ms as the reference reports them, plus
                   matvecs/s, algorithmic bytes and GB/s of one product;
* ``gpu_dense`` -- the exact O(N^2) sum on the GPU (``dense_matvec_gpu``);
* ``verify``    -- accuracy_rel_l2 of the gpu product against gpu_dense.

The reference's ``serial`` / ``parallel`` modes time its CPU executors and
are not part of this package (the CPU restatement lives in ``oracle/`` as
test infrastructure; ``bench.py --impl reference`` times it).  ``trace_out``
writes the per-kernel timeline of one product (in-kernel %globaltimer
records) as Chrome trace events in the reference's schema (metrics.py:67-84:
"X" events in microseconds, pid 1, tid = concurrent lane); ``csv_out``
writes ``mode,T_ms,matvecs_per_s``.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field

import numpy as np

from .geometry import CurveSpec, generate_sources
from .operators import NesaParams, build_tables
from .quadtree import TreeParams, build_tree, tree_stats

VALID_MODES = ("gpu", "gpu_dense", "verify")
CSV_HEADER = "mode,T_ms,matvecs_per_s"

KERNEL_TAGS = {
    1: "gather", 2: "scatter", 10: "near field (block GEMV)", 11: "reception (block GEMV, U)",
    20: "level up (leaf)", 21: "level up", 22: "level down", 30: "fused up (coarse levels)",
    31: "fused down (coarse levels)", 32: "sum children", 33: "translation reduce",
    40: "translation", 41: "translation (FFMA)", 42: "translation (tcgen05)",
    43: "translation (tcgen05, A in TMEM)", 44: "translation (tcgen05, persistent)",
    45: "translation (tcgen05, target-major)", 50: "level up (leaf, warp-tiled)",
    51: "level up (warp-tiled)", 52: "level down (warp-tiled)", 53: "level down + reception",
    54: "level down + beta", 60: "radiation (moments + A^)", 61: "radiation moments",
    70: "reception (expansion, beta in kernel)", 71: "reception (expansion)",
}


@dataclass(frozen=True)
class BenchConfig:
    n: int = 100_000
    p_avg: int = 50   # tree parameter P
    q_aux: int = 10   # equivalent sources per group, Q
    seed: int = 0
    curve: CurveSpec = field(default_factory=CurveSpec)
    modes: tuple[str, ...] = ("gpu",)
    repeats: int = 3
    part: str = "combined"  # combined | near | far
    dtype: str = "f32"      # operator / vector precision of the gpu mode
    complex_rhs: bool = True
    matvecs_per_sample: int = 20
    report_out: str | None = None
    trace_out: str | None = None
    csv_out: str | None = None

    def __post_init__(self):
        if self.n < 2:
            raise ValueError("n must be >= 2")
        if self.repeats < 1:
            raise ValueError("repeats must be >= 1")
        if self.matvecs_per_sample < 1:
            raise ValueError("matvecs_per_sample must be >= 1")
        for m in self.modes:
            if m not in VALID_MODES:
                raise ValueError(f"unknown mode {m!r}")
        if self.part not in ("combined", "near", "far"):
            raise ValueError("part must be combined, near or far")
        if self.dtype not in ("f32", "f64"):
            raise ValueError("dtype must be f32 or f64")


def _rhs(config: BenchConfig) -> np.ndarray:
    rng = np.random.default_rng(config.seed)
    if config.complex_rhs:
        re = rng.standard_normal(config.n)
        return re + 1j * rng.standard_normal(config.n)
    return rng.standard_normal(config.n)


def kernel_timeline(plan, q_ptr: int, phi_ptr: int, nrhs: int, is_complex: bool, near=True,
                    far=True, stream=None) -> list[dict]:
    """Per-kernel-launch spans of one product from the in-kernel records:
    [{name, grid, start_us, end_us}] relative to the first CTA start."""
    import torch
    lib = plan.lib
    cap = 1 << 16
    st = stream or torch.cuda.current_stream().cuda_stream
    lib.nesa_ktrace_enable(plan.handle, cap)
    try:
        plan.matvec_ptr(q_ptr, phi_ptr, nrhs, is_complex, near=near, far=far, stream=st)
        torch.cuda.synchronize()
        buf = (ctypes.c_uint64 * (4 * cap))()
        nrec = lib.nesa_ktrace_read(plan.handle, buf, cap)
    finally:
        lib.nesa_ktrace_enable(plan.handle, 0)
    rec = np.frombuffer(buf, dtype=np.uint64, count=4 * nrec).reshape(nrec, 4).astype(np.int64)
    if nrec == 0:
        return []
    t0 = rec[:, 2].min()
    spans: dict = {}
    for tag, grid, s, e in rec:
        k = (int(tag), int(grid))
        lo, hi = spans.get(k, (1 << 62, 0))
        spans[k] = (min(lo, s - t0), max(hi, e - t0))
    out = [{"name": KERNEL_TAGS.get(k[0], f"kernel {k[0]}"), "grid": k[1],
            "start_us": v[0] / 1e3, "end_us": v[1] / 1e3} for k, v in spans.items()]
    return sorted(out, key=lambda d: d["start_us"])


def timeline_to_chrome(spans: list[dict]) -> list[dict]:
    """Chrome trace events in the reference's schema (metrics.py:67-79);
    overlapping launches go to separate lanes (tid)."""
    lanes: list[float] = []
    events = []
    for sp in spans:
        for tid, end in enumerate(lanes):
            if end <= sp["start_us"]:
                break
        else:
            tid = len(lanes)
            lanes.append(0.0)
        lanes[tid] = sp["end_us"]
        events.append({"name": sp["name"], "ph": "X", "ts": sp["start_us"],
                       "dur": sp["end_us"] - sp["start_us"], "pid": 1, "tid": tid,
                       "args": {"grid": sp["grid"]}})
    return events


def run_benchmark(config: BenchConfig) -> dict:
    """Run the configured modes and return (and optionally write) a report.

    T_ms is the minimum over repeats of the mean product time of one sample
    (``matvecs_per_sample`` back-to-back graph launches timed with CUDA
    events on the launch stream, device-resident vectors); all samples are
    kept in the report.
    """
    import torch
    from .dense import dense_matvec_gpu
    from .fastmvp import task_counts
    from .plan import NesaPlan, algorithmic_bytes
    if not torch.cuda.is_available():
        raise RuntimeError("run_benchmark needs a CUDA device (no CPU fallback)")
    near = config.part in ("combined", "near")
    far = config.part in ("combined", "far")
    points = generate_sources(config.curve, config.n)
    q = _rhs(config)
    report: dict = {
        "config": {
            "n": config.n, "P": config.p_avg, "Q": config.q_aux, "seed": config.seed,
            "curve": config.curve.kind, "modes": list(config.modes), "repeats": config.repeats,
            "part": config.part, "dtype": config.dtype, "complex_rhs": config.complex_rhs,
            "matvecs_per_sample": config.matvecs_per_sample,
        },
    }
    phi_gpu = None
    spans = None
    if "gpu" in config.modes or "verify" in config.modes:
        tree = build_tree(points, TreeParams(P=config.p_avg))
        tables = build_tables(tree, NesaParams(Q=config.q_aux))
        report["tree_stats"] = tree_stats(tree)
        report["task_counts"] = task_counts(tree)
        plan = NesaPlan(tree, tables, dtype=config.dtype)
        cdt = {("f32", True): torch.complex64, ("f32", False): torch.float32,
               ("f64", True): torch.complex128, ("f64", False): torch.float64}[
            (config.dtype, config.complex_rhs)]
        qd = torch.from_numpy(q).to(cdt).cuda()
        phid = torch.empty_like(qd)
        st = torch.cuda.current_stream()
        run = lambda: plan.matvec_ptr(qd.data_ptr(), phid.data_ptr(), 1, config.complex_rhs,  # noqa: E731
                                      near=near, far=far, stream=st.cuda_stream)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        samples = []
        for _ in range(config.repeats):
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(st)
            for _ in range(config.matvecs_per_sample):
                run()
            t1.record(st)
            torch.cuda.synchronize()
            samples.append(t0.elapsed_time(t1) / config.matvecs_per_sample)
        t_ms = min(samples)
        R = 2 if config.complex_rhs else 1
        total = float(algorithmic_bytes(plan, R, near=near, far=far)["total"])
        report["gpu"] = {"samples_ms": samples, "T_ms": t_ms, "matvecs_per_s": 1e3 / t_ms,
                         "alg_bytes": total, "GB_s": total / (t_ms * 1e-3) / 1e9}
        spans = kernel_timeline(plan, qd.data_ptr(), phid.data_ptr(), 1, config.complex_rhs,
                                near=near, far=far, stream=st.cuda_stream)
        report["gpu"]["kernels"] = spans
        phi_gpu = phid.cpu().numpy().astype(np.complex128 if config.complex_rhs else np.float64)
        plan.close()
    dense_ref = None
    if "gpu_dense" in config.modes or "verify" in config.modes:
        samples = []
        for _ in range(config.repeats if "gpu_dense" in config.modes else 1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            dense_ref = dense_matvec_gpu(points, q)
            e1.record()
            torch.cuda.synchronize()
            samples.append(e0.elapsed_time(e1))
        if "gpu_dense" in config.modes:
            report["gpu_dense"] = {"samples_ms": samples, "T_ms": min(samples)}
    if "verify" in config.modes:
        report["accuracy_rel_l2"] = float(np.linalg.norm(phi_gpu - dense_ref) /
                                          np.linalg.norm(dense_ref))
    if config.report_out:
        with open(config.report_out, "w") as f:
            json.dump(report, f, indent=2)
    if config.trace_out and spans:
        with open(config.trace_out, "w") as f:
            json.dump(timeline_to_chrome(spans), f)
    if config.csv_out:
        with open(config.csv_out, "w") as f:
            f.write(CSV_HEADER + "\n")
            for m in ("gpu", "gpu_dense"):
                if m in report:
                    f.write(f"{m},{report[m]['T_ms']:.4f},{1e3 / report[m]['T_ms']:.2f}\n")
    return report
