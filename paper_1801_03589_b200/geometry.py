"""Source-point generators and bounding geometry (host side).

Mirrors the reference's ``taskfmm.geometry`` surface
(/root/reference/pkg/src/taskfmm/geometry.py:18-125): ``CurveSpec``,
``BBox``, ``parse_curve_spec``, ``generate_sources``, ``bounding_box`` with
the same kinds, argument meaning, determinism and ``ValueError`` behaviour.

It adds the 2D stand-ins for the BASELINE.json configurations (SURVEY.md
§8d, "Track A"): BASELINE asks for a sphere / ellipsoid+plates in 3D, the
reference only models 2D curves, so

* ``circle-random``  -- unit circle, angles drawn from ``default_rng(seed)``
  (C1/C2 analog of "uniform points on a unit sphere");
* ``ellipse-plates`` -- ellipse with semi-axes (5, 0.5), arc-length-uniform
  random points, plus two straight "plates" of length 4 at y = +-1.5;
  points split in proportion to length (C3/C4/C5 analog of the 10:1
  ellipsoid plus two 4x1 plates).

Plate placement is not fixed by BASELINE; the choice is documented in
DESIGN.md.  Right-hand sides are drawn by :func:`random_rhs` /
:func:`plane_wave_rhs` on a generator separate from the geometry's.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# Reference default wave curve x = t, y = A sin(2 pi f t), t in [0, 4]
# (geometry.py:9-13).
WAVE_AMPLITUDE = 0.35
WAVE_FREQUENCY = 1.5
WAVE_T_MAX = 4.0

# Analog geometry constants.
ELLIPSE_A = 5.0
ELLIPSE_B = 0.5
PLATE_LENGTH = 4.0
PLATE_OFFSET = 1.5

REFERENCE_KINDS = ("wave", "circle", "annulus-random")
CURVE_KINDS = REFERENCE_KINDS + ("circle-random", "ellipse-plates")


@dataclass(frozen=True)
class CurveSpec:
    """What curve the source points are sampled from (geometry.py:18-40)."""

    kind: str = "wave"
    amplitude: float = WAVE_AMPLITUDE
    frequency: float = WAVE_FREQUENCY
    radius: float = 1.0
    inner_radius: float = 1.0
    outer_radius: float = 2.0
    seed: int = 0

    def __post_init__(self):
        if self.kind not in CURVE_KINDS:
            raise ValueError(f"unknown curve kind {self.kind!r}")
        if self.kind == "wave" and self.amplitude <= 0:
            raise ValueError("wave amplitude must be positive")
        if self.kind in ("circle", "circle-random") and self.radius <= 0:
            raise ValueError("circle radius must be positive")
        if self.kind == "annulus-random" and not (
                0 < self.inner_radius < self.outer_radius):
            raise ValueError("annulus needs 0 < inner_radius < outer_radius")


@dataclass(frozen=True)
class BBox:
    """Axis-aligned bounding box (geometry.py:43-58)."""

    xmin: float
    ymin: float
    xmax: float
    ymax: float

    @property
    def extent(self) -> tuple[float, float]:
        return (self.xmax - self.xmin, self.ymax - self.ymin)

    @property
    def longest_side(self) -> float:
        return max(self.extent)


def parse_curve_spec(text: str, seed: int = 0) -> CurveSpec:
    """``"kind"`` or ``"kind:key=value,..."`` -> CurveSpec (geometry.py:61-76)."""
    kind, _, rest = text.partition(":")
    kwargs: dict = {}
    for item in filter(None, rest.split(",")) if rest else ():
        key, _, value = item.partition("=")
        if not value:
            raise ValueError(f"malformed curve parameter {item!r}")
        key = key.strip()
        kwargs[key] = int(value) if key == "seed" else float(value)
    kwargs.setdefault("seed", seed)
    return CurveSpec(kind=kind.strip(), **kwargs)


def _ellipse_arclength_table(a: float, b: float, n_tab: int = 1 << 16):
    """Cumulative arc length s(t) of (a cos t, b sin t) on a uniform t grid."""
    t = np.linspace(0.0, 2.0 * np.pi, n_tab + 1)
    speed = np.hypot(a * np.sin(t), b * np.cos(t))
    s = np.concatenate(([0.0], np.cumsum(0.5 * (speed[1:] + speed[:-1]) * np.diff(t))))
    return t, s


def ellipse_perimeter(a: float = ELLIPSE_A, b: float = ELLIPSE_B) -> float:
    return float(_ellipse_arclength_table(a, b)[1][-1])


def _ellipse_plates(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    t_tab, s_tab = _ellipse_arclength_table(ELLIPSE_A, ELLIPSE_B)
    perim = s_tab[-1]
    total = perim + 2.0 * PLATE_LENGTH
    n_e = int(round(n * perim / total))
    n_top = (n - n_e) // 2
    n_bot = n - n_e - n_top
    u = rng.random(n_e) * perim
    t = np.interp(u, s_tab, t_tab)
    ell = np.column_stack((ELLIPSE_A * np.cos(t), ELLIPSE_B * np.sin(t)))
    xt = -0.5 * PLATE_LENGTH + PLATE_LENGTH * rng.random(n_top)
    xb = -0.5 * PLATE_LENGTH + PLATE_LENGTH * rng.random(n_bot)
    top = np.column_stack((xt, np.full(n_top, PLATE_OFFSET)))
    bot = np.column_stack((xb, np.full(n_bot, -PLATE_OFFSET)))
    return np.concatenate((ell, top, bot))


def generate_sources(spec: CurveSpec, n: int) -> np.ndarray:
    """n source points (n, 2) float64; bit-identical for a given (spec, n).

    The three reference kinds follow geometry.py:79-115 exactly; the
    analog kinds are described in the module docstring.
    """
    if n < 2:
        raise ValueError("need at least 2 source points")
    if spec.kind == "wave":
        t = WAVE_T_MAX * (np.arange(n) + 0.5) / n          # midpoint rule
        pts = np.column_stack(
            (t, spec.amplitude * np.sin(2.0 * np.pi * spec.frequency * t)))
    elif spec.kind == "circle":
        theta = 2.0 * np.pi * np.arange(n) / n
        pts = spec.radius * np.column_stack((np.cos(theta), np.sin(theta)))
    elif spec.kind == "annulus-random":
        rng = np.random.Generator(np.random.Philox(spec.seed))
        u = rng.random((n, 2))
        r = np.sqrt(spec.inner_radius ** 2
                    + u[:, 0] * (spec.outer_radius ** 2 - spec.inner_radius ** 2))
        theta = 2.0 * np.pi * u[:, 1]
        pts = np.column_stack((r * np.cos(theta), r * np.sin(theta)))
    elif spec.kind == "circle-random":
        theta = 2.0 * np.pi * np.random.default_rng(spec.seed).random(n)
        pts = spec.radius * np.column_stack((np.cos(theta), np.sin(theta)))
    else:  # ellipse-plates
        pts = _ellipse_plates(n, spec.seed)

    if not np.isfinite(pts).all():
        raise ValueError("generated non-finite coordinates")
    if np.unique(pts, axis=0).shape[0] != n:
        raise ValueError("generated coincident points; change n or seed")
    return pts


def bounding_box(points: np.ndarray) -> BBox:
    """Tight box around (n, 2) points (geometry.py:118-125)."""
    points = np.asarray(points, dtype=float)
    if points.ndim != 2 or points.shape[1] != 2 or points.shape[0] == 0:
        raise ValueError("points must be a nonempty (n, 2) array")
    lo = points.min(axis=0)
    hi = points.max(axis=0)
    return BBox(lo[0], lo[1], hi[0], hi[1])


def curve_length(spec: CurveSpec) -> float:
    """Arc length of the curve (for the 10-points-per-wavelength k)."""
    if spec.kind == "wave":
        t = np.linspace(0.0, WAVE_T_MAX, (1 << 16) + 1)
        dy = spec.amplitude * 2 * np.pi * spec.frequency * np.cos(
            2 * np.pi * spec.frequency * t)
        sp = np.hypot(1.0, dy)
        return float(np.sum(0.5 * (sp[1:] + sp[:-1]) * np.diff(t)))
    if spec.kind in ("circle", "circle-random"):
        return 2.0 * math.pi * spec.radius
    if spec.kind == "ellipse-plates":
        return ellipse_perimeter() + 2.0 * PLATE_LENGTH
    raise ValueError("curve length undefined for an area distribution")


def wavenumber(spec: CurveSpec, n: int, points_per_wavelength: float = 10.0) -> float:
    """k = 2 pi / lambda with lambda = ppw * (arc length / n)."""
    h = curve_length(spec) / n
    return 2.0 * math.pi / (points_per_wavelength * h)


def random_rhs(n: int, seed: int, complex_: bool = True) -> np.ndarray:
    """q = N(0,1) + 1j N(0,1) (real part first) from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    re = rng.standard_normal(n)
    if not complex_:
        return re
    return re + 1j * rng.standard_normal(n)


def plane_wave_rhs(points: np.ndarray, k: float, n_waves: int = 64) -> np.ndarray:
    """(n, n_waves) complex128: q_m = exp(-1j k d_m . r), phi_m = 2 pi m / n_waves."""
    ang = 2.0 * np.pi * np.arange(n_waves) / n_waves
    d = np.stack((np.cos(ang), np.sin(ang)))            # (2, M)
    return np.exp(-1j * k * (points @ d))
