"""bench.py's output contract, checked on CPU with the reference arm (the
oracle port of mvp_serial, whole products; the only arm that runs without a
GPU)."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--n", "20000", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "matvecs/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert "workload" in d["config"]
    # whole products, and the product library never loaded in this process
    assert d["native_libs_loaded"] == []
    assert d["step_s"]["min"] > 0 and d["task_parallel"]["value"] > 0


import pytest  # noqa: E402


@pytest.mark.gpu
def test_bench_json_line_on_gpu():
    # the full arm at a reduced size: every key of the contract, the roofline
    # and end-to-end objects, clocks and the launch count
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--n", "200000", "--steps", "20",
                          "--warmup", "3"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 200000 * 8 and e["d2h_bytes_per_step"] == 200000 * 8
    assert d["gpu_launches"] == d["steps"] * d["gpu_launches"] // d["steps"] > 0
    assert d["clocks"]["sm_mhz"] > 0 and d["cpu_baseline"]["value"] > 0
    # the extra configurations: C5 (64 right-hand sides) and Track B (3D Helmholtz)
    assert d["c5"]["far_field_gemms"] and d["c5"]["ms_per_64rhs_product"] > 0
    assert d["track_b"]["us_per_product"] > 0
