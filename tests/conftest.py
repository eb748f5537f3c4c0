"""pytest configuration: `gpu` marker, repo on sys.path, golden loader."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: takes more than ~20 s on CPU")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


GOLDEN_CASES = ["fastmvp_1500", "grid4_single_level", "wave_3000_P50_Q10", "annulus_1024",
                "c1_wave_2000", "c1_circle_2000", "c2_circle_20000", "c2_wave_20000",
                "ellipse_plates_20000"]


def grid_points(k: int) -> np.ndarray:
    c = (np.arange(k) + 0.5) / k
    xx, yy = np.meshgrid(c, c)
    return np.column_stack((xx.ravel(), yy.ravel()))


def have_reference() -> bool:
    return os.path.isdir(REFERENCE_SRC)


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]
    return get
