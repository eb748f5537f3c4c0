#!/usr/bin/env python
"""Benchmark: NESA matvecs/s at N = 2M on 1..8 B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[3], "C4"), Track A 2D analog:
N = 2,000,000 points on the ellipse+plates union (seed 3), leaf target P = 64,
Q = 64 equivalent sources, complex64 right-hand side (N(0,1) + 1j N(0,1),
seed 3, separate generator), float32 operators.  One step = one full product
phi = K~ q (gather, near field, radiation, upward, translation, downward,
reception, scatter).  Inputs stay resident in HBM for ``value``; ``e2e``
goes through the public API (paper_1801_03589_b200.mvp) with pinned host
buffers, host<->device copies inside the timed region.

``--impl reference`` times the reference's CPU algorithm -- the oracle port
(oracle/mvp_oracle.py, the restated taskfmm mvp_serial; the reference itself
is pure Python and not present on the GPU box) -- one WHOLE complex product
per step (Re and Im as two real calls), on the host's cores, in a process
that never loads the product library; plus one product of the reference's
task-parallel form (oracle/task_mvp.py).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

N_POINTS = 2_000_000
SEED = 3
LEAF_P = 64
Q_AUX = 64
METRIC = "NESA matvecs/sec at N=2M (1/2/4/8 B200); achieved HBM GB/s vs roofline"
UNIT = "matvecs/s"


def workload_config(n=N_POINTS, world=1):
    return {
        "workload": f"C4 2D analog: ellipse(5,0.5)+2 plates, N={n:,}, seed {SEED}, "
                    f"leaf P={LEAF_P}, Q={Q_AUX}, complex64 rhs, float32 operators",
        "N": n, "P": LEAF_P, "Q": Q_AUX, "geometry": "ellipse-plates", "seed": SEED,
        "vectors": "complex64", "operators": "float32",
        "parallelism": f"morton-partition x{world}" if world > 1 else "single-gpu",
        "l2": "no flush needed: each step streams the 2.13 GB near-field operator (> 126 MB L2)",
    }


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_POINTS, help="points (default 2M)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-task-form", action="store_true",
                    help="reference arm: skip the task-parallel form's timing")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c128", action="store_true", help="skip the complex128 product timing")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the C5 (64 right-hand sides) and Track B (3D Helmholtz) timings")
    ap.add_argument("--pipe-slots", type=int, default=1,
                    help="compute slots of the pipelined e2e API (independent plans)")
    return ap.parse_args(argv)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def build_problem(n):
    import paper_1801_03589_b200 as nesa
    t0 = time.perf_counter()
    pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=SEED), n)
    t1 = time.perf_counter()
    tree = nesa.build_tree(pts, nesa.TreeParams(P=LEAF_P))
    t2 = time.perf_counter()
    params = nesa.NesaParams(Q=Q_AUX)
    tables = nesa.build_tables(tree, params)
    t3 = time.perf_counter()
    q = nesa.random_rhs(n, SEED).astype(np.complex64)
    return pts, tree, params, tables, q, {"points_s": t1 - t0, "tree_s": t2 - t1,
                                          "tables_s": t3 - t2}


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except (OSError, ValueError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r)
                          if v.lower().startswith("active")})
        sm = [r[0] for r in rows]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def load_peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic():
    """dram bytes/launch of the near kernel from the committed ncu capture."""
    p = os.path.join(HERE, "profiles", "ncu_near_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle port of the reference's product
# ---------------------------------------------------------------------------
def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def reference_problem(n):
    """Tree and OperatorSet exactly as the reference builds them, on the host,
    WITHOUT the product library: the numpy tree restatement (bit-identical to
    the reference's build_tree, tests/test_host_tree.py) and the host operator
    assembly (build_all, pinned to the reference's checksums)."""
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.quadtree import build_tree
    pts = nesa.generate_sources(nesa.CurveSpec(kind="ellipse-plates", seed=SEED), n)
    t0 = time.perf_counter()
    tree = build_tree(pts, nesa.TreeParams(P=LEAF_P), native=False)
    params = nesa.NesaParams(Q=Q_AUX)
    ops = nesa.build_all(tree, params)
    q = nesa.random_rhs(n, SEED).astype(np.complex64)
    return tree, ops, q, time.perf_counter() - t0


def reference_product(tree, ops, q):
    """One complex product as the reference computes it: mvp_serial on Re q
    and on Im q (float64; the operator is real)."""
    from oracle.mvp_oracle import mvp_serial
    t0 = time.perf_counter()
    mvp_serial(tree, ops, q.real.astype(np.float64))
    mvp_serial(tree, ops, q.imag.astype(np.float64))
    return time.perf_counter() - t0


def reference_task_product(tree, ops, q, workers):
    """The reference's task-parallel form (mvp with a Runtime of `workers`
    threads, fastmvp.py:124-139), restated in oracle/task_mvp.py."""
    from oracle.task_mvp import TaskRuntime, mvp_tasks
    with TaskRuntime(workers) as rt:
        t0 = time.perf_counter()
        mvp_tasks(tree, ops, q.real.astype(np.float64), rt)
        mvp_tasks(tree, ops, q.imag.astype(np.float64), rt)
        return time.perf_counter() - t0


def loaded_native_libs():
    try:
        return sorted({ln.split()[-1] for ln in open("/proc/self/maps") if "libnesa" in ln})
    except OSError:
        return []


def run_cpu_baseline(tree_unused, n, repeats=2):
    """cpu_baseline of our arm: whole complex products of the oracle port at
    the bench workload, min of `repeats`."""
    tree, ops, q, build_s = reference_problem(n)
    ts = [reference_product(tree, ops, q) for _ in range(repeats)]
    t = min(ts)
    return {"value": 1.0 / t, "unit": UNIT, "cores": cpu_threads(), "kind": "port",
            "sample": f"whole products at N={n:,}: oracle port of taskfmm mvp_serial "
                      f"(fastmvp.py:142-172), float64, complex q as two real calls (Re, Im); "
                      f"min of {repeats}: {t:.3f} s per product (all {len(ts)}: "
                      f"{', '.join(f'{x:.3f}' for x in ts)} s); host build {build_s:.1f} s untimed",
            "seconds_per_product": t, "cpu_model": cpu_model()}


def run_reference(args):
    """--impl reference: the reference's CPU product (the oracle port; the
    reference is pure Python and absent on the GPU box) on the host cores,
    every step one WHOLE complex product of the bench workload.  This process
    never loads libnesa_b200.so (checked and reported)."""
    rank, _, world = dist_env()
    if world > 1 and rank != 0:
        return
    tree, ops, q, build_s = reference_problem(args.n)
    for _ in range(args.warmup):
        reference_product(tree, ops, q)
    times = [reference_product(tree, ops, q) for _ in range(args.steps)]
    tot = float(np.sum(times))
    value = args.steps / tot
    workers = os.cpu_count() or 1
    t_task = reference_task_product(tree, ops, q, workers) if not args.no_task_form else None
    cores = cpu_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.n, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": "every step one whole complex product at the bench workload: "
                                   "oracle port of taskfmm mvp_serial (fastmvp.py:142-172, "
                                   "float64, Re and Im as two real calls, numpy/OpenBLAS on all "
                                   "host threads)",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_s": {"min": float(np.min(times)), "median": float(np.median(times)),
                   "max": float(np.max(times))},
        "task_parallel": None if t_task is None else {
            "value": 1.0 / t_task, "unit": UNIT, "workers": workers, "seconds_per_product": t_task,
            "form": "reference mvp(tree, ops, q, Runtime(RuntimeConfig(workers=os.cpu_count()))) "
                    "restated in oracle/task_mvp.py (fastmvp.py:124-139, runtime.py); one whole "
                    "complex product; GIL-bound as in BASELINE.md §2"},
        "host_build_s": build_s,
        "native_libs_loaded": loaded_native_libs(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def time_c128(args, tree, tables, q, dev, stream):
    """complex128 products with a float64 plan (BASELINE north_star's 1e-12
    precision), timed like the headline: CUDA events around K graph launches,
    device-resident q / phi; plus the near kernel's in-graph roofline."""
    import torch
    from paper_1801_03589_b200.plan import NesaPlan, algorithmic_bytes
    plan = NesaPlan(tree, tables, dtype="f64", device=dev.index)
    qd = torch.from_numpy(q.astype(np.complex128)).to(dev)
    phid = torch.empty_like(qd)

    def step(profile=False):
        plan.matvec_ptr(qd.data_ptr(), phid.data_ptr(), 1, True, stream=stream.cuda_stream,
                        profile="near" if profile else False)

    def timed(profile):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step(profile)
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / args.steps

    for _ in range(max(args.warmup, 3)):
        step()
        step(True)
    for _ in range(args.steps):  # grow the profiling event pool to K (untimed)
        step(True)
    torch.cuda.synchronize()
    plan.profile_reset()
    ms = timed(False)            # the number (plain products)
    timed(True)                  # the near kernel's in-graph duration (event nodes)
    near_ms = float(np.mean(plan.profile_read("near")))
    alg = algorithmic_bytes(plan, 2)
    peak, _ = load_peaks()
    out = {"value": 1e3 / ms, "unit": UNIT, "ms_per_step": ms, "steps": args.steps,
           "dtype": "c128", "operators": "float64",
           "near_roofline": {"achieved": alg["near"] / (near_ms * 1e-3) / 1e9, "peak": peak,
                             "frac": alg["near"] / (near_ms * 1e-3) / 1e9 / peak,
                             "avg_launch_ms": near_ms, "alg_bytes_per_launch": alg["near"]},
           "matvec_alg_bytes": alg["total"], "matvec_achieved_gbs": alg["total"] / (ms * 1e-3) / 1e9,
           "gpu_launches": plan.stat("kernels_per_matvec") * args.steps}
    plan.close()
    del qd, phid
    torch.cuda.empty_cache()
    return out


def _time_events(fn, steps, stream):
    import torch
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def time_c5(args, dev, stream):
    """BASELINE configs[4] (2D analog): 200k points (ellipse + plates, seed 4),
    64 plane-wave right-hand sides = 128 real columns, leaf P = 64, Q = 48,
    complex64: one product of all 64 columns (near field as one tensor-core
    GEMM, far field as batched GEMMs over the 128 columns)."""
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.plan import NesaPlan
    n, P, Qa = 200_000, 64, 48
    spec = nesa.CurveSpec(kind="ellipse-plates", seed=4)
    pts = nesa.generate_sources(spec, n)
    Qm = nesa.plane_wave_rhs(pts, nesa.wavenumber(spec, n), 64).astype(np.complex64)
    tree = nesa.build_tree(pts, nesa.TreeParams(P=P))
    plan = NesaPlan(tree, nesa.build_tables(tree, nesa.NesaParams(Q=Qa)), dtype="f32",
                    device=dev.index, stored_vu=True)
    qd = torch.from_numpy(np.ascontiguousarray(Qm)).to(dev)
    phid = torch.empty_like(qd)

    def step():
        plan.matvec_ptr(qd.data_ptr(), phid.data_ptr(), 64, True, stream=stream.cuda_stream)

    for _ in range(3):
        step()
    ms = _time_events(step, 20, stream)
    out = {"workload": f"C5 2D analog: N={n:,}, seed 4, leaf P={P}, Q={Qa}, 64 plane waves "
                       "(complex64, 128 real columns)",
           "ms_per_64rhs_product": ms, "rhs_per_s": 64e3 / ms, "products_64rhs_per_s": 1e3 / ms,
           "far_field_gemms": plan.stat("far_wide") == 1, "near_tensor_core_gemm": plan.stat("near_wide") == 1}
    plan.close()
    del qd, phid
    torch.cuda.empty_cache()
    return out


def time_track_b(args, dev, stream):
    """Track B: BASELINE configs[2] literally -- 200k points on the 3D
    ellipsoid (5, 0.5, 0.5) + two 4 x 1 plates (seed 2), octree leaf P = 48,
    Q = 48, Helmholtz kernel at 10 points per wavelength, complex operators,
    complex64 vectors (float32 engine)."""
    import torch
    from paper_1801_03589_b200 import helmholtz as hz
    from paper_1801_03589_b200.plan3 import HelmholtzPlan
    t0 = time.perf_counter()
    pts, tree, params, q = hz.track_b_problem("ellipsoid-plates", 200_000, 2, 48, 48)
    plan = HelmholtzPlan(tree, hz.build_tables3(tree, params), "c64", device=dev.index)
    build_s = time.perf_counter() - t0
    qd = torch.from_numpy(q.astype(np.complex64)).to(dev)
    xr = torch.view_as_real(qd.reshape(-1, 1)).permute(0, 2, 1).contiguous()
    yr = torch.empty_like(xr)

    def step():
        plan.matvec_ptr(xr.data_ptr(), yr.data_ptr(), 1, False, stream=stream.cuda_stream)

    for _ in range(3):
        step()
    ms = _time_events(step, 50, stream)
    near_bytes = plan.stat("near_entries") * 4
    out = {"workload": f"Track B C3: N=200,000 3D ellipsoid+plates, seed 2, octree leaf P=48, Q=48, "
                       f"Helmholtz k={params.k:.2f}, complex64",
           "us_per_product": ms * 1e3, "products_per_s": 1e3 / ms,
           "near_bytes": near_bytes, "near_bytes_per_s_over_product": near_bytes / (ms * 1e-3),
           "levels": tree.L - tree.l0 + 1, "host_build_s": build_s}
    plan.close()
    del qd, xr, yr
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# (our arm)
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import paper_1801_03589_b200 as nesa
    from paper_1801_03589_b200.plan import NesaPlan, algorithmic_bytes

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    pts, tree, params, tables, q, build_t = build_problem(args.n)
    t0 = time.perf_counter()
    if world > 1:
        from paper_1801_03589_b200.dist import DistNesa
        engine = DistNesa(tree, tables, dtype="f32", device=local_rank)
        plan = engine.plan
    else:
        engine = None
        plan = NesaPlan(tree, tables, dtype="f32", device=local_rank)
    torch.cuda.synchronize()
    build_t["plan_s"] = time.perf_counter() - t0

    qd = torch.from_numpy(q).to(dev)
    phid = torch.empty_like(qd)
    stream = torch.cuda.current_stream(dev)

    def step(profile=False):
        if engine is not None:
            # one graph per rank: the halo exchange (NCCL all_gather) is inside
            engine.matvec_ptr(qd.data_ptr(), phid.data_ptr(), 1, True, stream=stream.cuda_stream,
                              profile="near" if profile else False)
        else:
            plan.matvec_ptr(qd.data_ptr(), phid.data_ptr(), 1, True, stream=stream.cuda_stream,
                            profile="near" if profile else False)

    prof = True
    for _ in range(max(args.warmup, 3)):
        step()
        step(prof)
    # soak clocks ~1 s, then grow the profiling event pool to K (untimed)
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    sampler.start()
    t_soak = time.perf_counter()
    n_soak = 0
    while time.perf_counter() - t_soak < 1.0:
        step()
        n_soak += 1
        if n_soak % 50 == 0:
            torch.cuda.synchronize()
    if prof:
        plan.profile_reset()
        for i in range(args.steps):
            step(prof)
            if i % 50 == 49:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        plan.profile_reset()

    def timed(profile):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            step(profile)
        ev1.record(stream)
        ev1.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # timed region 1 (the headline): K plain products.  Timed region 2: the
    # same K products with two event-record nodes around the near-field
    # kernel on its own stream (the roofline's in-graph duration).  The event
    # nodes need a per-launch graph update (cudaGraphExecEventRecordNodeSetEvent)
    # that costs ~19 us per product (tools/ab.py ... :AB_PROFILE=1, 502.8 vs
    # 521.9 us), so the headline does not carry them.
    ms = timed(False)
    ms_prof = timed(True) if prof else None
    clocks = sampler.stop()
    ms_step = ms / args.steps
    value = 1e3 / ms_step            # whole-job products per second (strong scaling)

    # roofline of the dominant kernel (near field), from the in-graph events
    alg = algorithmic_bytes(plan, 2)
    roofline = None
    stages = {}
    if prof:
        for st in ("near",):   # only the near-field events are in the timed graph
            d = plan.profile_read(st)
            stages[st] = float(np.mean(d)) if d.size else None
        near_ms = stages["near"]
        peak, peak_src = load_peaks()
        near_bytes = alg["near"]
        ach = near_bytes / (near_ms * 1e-3) / 1e9
        traffic = load_traffic()
        roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                    "frac": ach / peak,
                    "traffic": traffic.get("bytes_per_launch") if traffic else None,
                    "kernel": "blockgemv_kernel<float,2,store> (near field)",
                    "alg_bytes_per_launch": near_bytes, "avg_launch_ms": near_ms,
                    "peak_source": peak_src,
                    "timed_region": {"steps": args.steps, "ms_per_step": ms_prof / args.steps,
                                     "note": "second timed region: the same K products with CUDA "
                                             "events around the near kernel on its stream"},
                    "note": "near kernel inside the full product, concurrent with the radiation "
                            "and far-field chain (they share HBM and SMs)"
                            + (f"; rank {rank} of {world}, its own leaves" if world > 1 else "")}
        if world > 1:
            # per-rank figures (each rank streams its own leaves' operator)
            t = torch.tensor([ach, near_ms], device=dev, dtype=torch.float64)
            allr = [torch.zeros_like(t) for _ in range(world)]
            torch.distributed.all_gather(allr, t)
            roofline["per_rank"] = [{"rank": i, "achieved": float(x[0]), "frac": float(x[0]) / peak,
                                     "avg_launch_ms": float(x[1])} for i, x in enumerate(allr)]
        # the same kernel with nothing concurrent (near-only product), for context
        for _ in range(5 if world == 1 else 0):
            plan.matvec_ptr(qd.data_ptr(), phid.data_ptr(), 1, True, far=False,
                            stream=stream.cuda_stream, profile="near")
        if world == 1:
            plan.profile_reset()
            for _ in range(50):
                plan.matvec_ptr(qd.data_ptr(), phid.data_ptr(), 1, True, far=False,
                                stream=stream.cuda_stream, profile="near")
            torch.cuda.synchronize()
            iso = float(np.mean(plan.profile_read("near")))
            roofline["isolated"] = {"achieved": near_bytes / (iso * 1e-3) / 1e9,
                                    "frac": near_bytes / (iso * 1e-3) / 1e9 / peak,
                                    "avg_launch_ms": iso,
                                    "note": "near-only product, nothing concurrent"}
    matvec_bw = alg["total"] / (ms_step * 1e-3) / 1e9

    # the reference's own precision: a complex128 product (float64 plan,
    # operators assembled on the device as for the headline), same workload
    c128 = None
    if world == 1 and not args.no_c128:
        c128 = time_c128(args, tree, tables, q, dev, stream)

    # end to end through the public API with pinned host buffers: the
    # pipelined API (H2D of step k+1 and D2H of step k-1 overlap product k;
    # every step still uploads its q and downloads its phi), and the
    # synchronous mvp() call for reference
    e2e = None
    if not args.no_e2e and world == 1:
        qh = torch.from_numpy(q).pin_memory()
        k2 = max(10, min(args.steps, 100))
        pipe = nesa.MvpPipeline(tree, tables, dtype="f32", is_complex=True,
                                slots=args.pipe_slots)
        outs = [torch.empty_like(qh).pin_memory() for _ in range(2)]
        for i in range(4):
            pipe.submit(qh, outs[i % 2])
        pipe.synchronize()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(pipe.s_h2d)
        for i in range(k2):
            pipe.submit(qh, outs[i % 2])
        e1.record(pipe.s_d2h)
        e1.synchronize()
        e_ms = e0.elapsed_time(e1) / k2
        # synchronous call
        for _ in range(3):
            nesa.mvp(tree, tables, qh)
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(k2):
            out = nesa.mvp(tree, tables, qh)
        s1.record(stream)
        s1.synchronize()
        s_ms = s0.elapsed_time(s1) / k2
        e2e = {"value": 1e3 / e_ms, "unit": UNIT, "h2d_bytes_per_step": int(qh.numel() * 8),
               "d2h_bytes_per_step": int(out.numel() * 8), "ms_per_step": e_ms,
               "api": f"paper_1801_03589_b200.MvpPipeline(tree, tables, slots={args.pipe_slots})"
                      ".submit(pinned q, pinned phi) x K, synchronize(): every step uploads its q "
                      "and downloads its phi; transfers and the products of neighbouring "
                      "(independent) steps overlap",
               "slots": args.pipe_slots,
               "sync_call": {"value": 1e3 / s_ms, "ms_per_step": s_ms,
                             "api": "paper_1801_03589_b200.mvp(tree, tables, pinned torch.complex64 (N,))"}}

    if not args.no_e2e and world > 1:
        # every rank: its q (the full vector, original order) from pinned host
        # memory, the distributed product, its phi back (its points' entries;
        # the ranks' outputs are disjoint); time = max over ranks
        qh = torch.from_numpy(q).pin_memory()
        ph = torch.empty_like(qh).pin_memory()
        qd2 = torch.empty_like(qd)
        phd2 = torch.zeros_like(qd)
        k2 = max(10, min(args.steps, 100))

        def e2e_step():
            qd2.copy_(qh, non_blocking=True)
            engine.matvec_ptr(qd2.data_ptr(), phd2.data_ptr(), 1, True, stream=stream.cuda_stream)
            ph.copy_(phd2, non_blocking=True)

        for _ in range(3):
            e2e_step()
        torch.cuda.synchronize()
        torch.distributed.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k2):
            e2e_step()
        e1.record(stream)
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / k2], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e_ms = float(t.item())
        e2e = {"value": 1e3 / e_ms, "unit": UNIT, "h2d_bytes_per_step": int(qh.numel() * 8) * world,
               "d2h_bytes_per_step": int(ph.numel() * 8) * world, "ms_per_step": e_ms,
               "api": "paper_1801_03589_b200.dist.DistNesa.matvec_ptr per rank: H2D of q from pinned "
                      "memory, product (one graph: near field || radiation + upward pass, NCCL "
                      "all_gather of partial source amplitudes, translation + downward pass, "
                      "reception), D2H of the rank's phi; max over ranks"}

    c5 = track_b = None
    if world == 1 and not args.no_extras:
        c5 = time_c5(args, dev, stream)
        track_b = time_track_b(args, dev, stream)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baseline(tree, args.n)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c64", "data": "synthetic (seeded ellipse+plates geometry, N(0,1) rhs)",
            "config": workload_config(args.n, world),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "c128": c128,
            "c5": c5, "track_b": track_b,
            "gpu_launches": plan.stat("kernels_per_matvec") * args.steps,
            "clocks": clocks,
            "matvec_alg_bytes": alg["total"], "matvec_achieved_gbs": matvec_bw,
            "stage_ms": stages, "build_s": build_t,
            "plan": {"near_entries": plan.stat("near_entries"),
                     "v_entries": plan.stat("v_entries"), "d_refs": plan.stat("d_refs"),
                     "n_dtab": plan.stat("n_dtab"), "levels": tree.L - tree.l0 + 1,
                     "groups": tree.arrays.n_groups, "leaves": tree.n_leaves,
                     "device_bytes": plan.stat("device_bytes")},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main(argv=None):
    args = parse_args(argv)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
