"""Host-side value types of the hot path's interface.

These mirror the reference's dataclasses field for field so the drop-in
entry points accept and return the same shapes of data:

  IntensityImage / RampedImage      imaging.py:28-63
  ScaleSet / FeaturePoint           detector.py:33-80
  DescriptorConfig / DescribedFeatures  descriptor.py:37-79
  MatcherConfig / MatchPair         matcher.py:16-36
  RigidTransform / RansacConfig / RegistrationResult  registration.py:27-97

Objects of the reference package itself are accepted everywhere too (the
entry points only read attributes).  Nothing in this module computes on the
hot path; the GPU work lives in ``device.py`` and the C-ABI library.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from .errors import ConfigError

MIN_WINDOW = 8
POLARITY_MAX, POLARITY_MIN = "max", "min"
STRATEGY_NEAREST, STRATEGY_THRESHOLD_ALL = "nearest_neighbor", "threshold_all"
STRATEGY_RATIO = "ratio_test"  # extra strategy (not in the reference): Lowe ratio, MatcherConfig.ratio
ORIENTATION_BINS, PEAK_BINS = 8, 36
TWO_PI = 2.0 * math.pi
RAMP_SPAN_LIMIT = 0.05 * 255.0


# ---- images -------------------------------------------------------------------

@dataclass(frozen=True, eq=False)
class IntensityImage:
    """Grayscale raster (numpy array or torch tensor, CPU or CUDA)."""

    pixels: object
    image_id: str = ""

    def __post_init__(self):
        shape = tuple(self.pixels.shape)
        if len(shape) != 2 or shape[0] * shape[1] == 0:
            raise ValueError("pixels must be a non-empty 2-D array")

    @property
    def nr(self) -> int:
        return int(self.pixels.shape[0])

    @property
    def nc(self) -> int:
        return int(self.pixels.shape[1])


@dataclass(frozen=True, eq=False)
class RampedImage:
    """Ramped raster.  Built by ``apply_linear_ramp`` it keeps the raw pixels
    and alpha so the GPU recomputes the ramp bit-exactly on the fly; the
    float64 ``pixels`` view is materialised on the host only on request."""

    pixels: object
    alpha: float
    source_id: str = ""
    raw: object = None

    @property
    def nr(self) -> int:
        return int((self.raw if self.raw is not None else self.pixels).shape[0])

    @property
    def nc(self) -> int:
        return int((self.raw if self.raw is not None else self.pixels).shape[1])


class _LazyRamp:
    """Host float64 view of raw + ramp, computed on first use."""

    def __init__(self, raw, alpha):
        self._raw, self._alpha, self._val = raw, alpha, None
        self.shape = tuple(raw.shape)
        self.ndim = 2

    def _get(self):
        if self._val is None:
            raw = self._raw.cpu().numpy() if hasattr(self._raw, "cpu") else np.asarray(self._raw)
            nr, nc = raw.shape
            k = np.arange(1, nr * nc + 1, dtype=np.float64).reshape(nr, nc)
            self._val = raw.astype(np.float64) + k * self._alpha
        return self._val

    def __array__(self, dtype=None, copy=None):
        v = self._get()
        return v if dtype is None else v.astype(dtype)

    def __getitem__(self, item):
        return self._get()[item]


def default_alpha(nr: int, nc: int) -> float:
    """imaging.py:108-111."""
    return 1e-6 * 255.0 / (nr * nc)


def apply_linear_ramp(img: IntensityImage, alpha: float) -> RampedImage:
    """imaging.py:113-132; validation identical, ramp deferred to the device."""
    if not math.isfinite(alpha) or alpha <= 0:
        raise ConfigError(f"alpha must be positive, got {alpha}")
    if alpha * img.nr * img.nc > RAMP_SPAN_LIMIT:
        raise ConfigError(
            f"alpha={alpha} spans {alpha * img.nr * img.nc:.3g} intensity levels over "
            f"{img.nr}x{img.nc}; limit is {RAMP_SPAN_LIMIT}")
    return RampedImage(pixels=_LazyRamp(img.pixels, alpha), alpha=alpha, source_id=img.image_id,
                       raw=img.pixels)


# ---- detection ------------------------------------------------------------------

class Window(NamedTuple):
    row0: int
    col0: int
    height: int
    width: int


@dataclass(frozen=True)
class ScaleSet:
    """Strictly increasing window sides, each >= 8 (detector.py:33-68)."""

    sizes: tuple

    def __post_init__(self):
        if not self.sizes:
            raise ConfigError("scale set must contain at least one size")
        if any(int(s) != s or s < MIN_WINDOW for s in self.sizes):
            raise ConfigError(f"window sizes must be integers >= {MIN_WINDOW}")
        if any(b <= a for a, b in zip(self.sizes, self.sizes[1:])):
            raise ConfigError("window sizes must be strictly increasing")

    @property
    def l_max(self) -> int:
        return self.sizes[-1]

    @classmethod
    def from_range(cls, l_min: int, l_max: int) -> "ScaleSet":
        if l_min > l_max:
            raise ConfigError(f"window range [{l_min}, {l_max}] is empty")
        out, s = [], int(l_min)
        while s < l_max:
            out.append(s)
            s *= 2
        return cls(tuple(out + [int(l_max)]))

    def validate_for(self, nr: int, nc: int) -> None:
        if self.l_max > min(nr, nc):
            raise ConfigError(f"largest window {self.l_max} exceeds image side {min(nr, nc)}")


@dataclass(frozen=True)
class FeaturePoint:
    row: int
    col: int
    scale: int
    polarity: str
    window_index: int
    value: float


def window_count(nr: int, nc: int, size: int) -> int:
    return -(-nr // size) * (-(-nc // size))


def partition_windows(nr: int, nc: int, size: int) -> list:
    """Row-major tiling with shrunk trailing windows (detector.py:87-103)."""
    if size < MIN_WINDOW or size > min(nr, nc):
        raise ConfigError(f"window size {size} outside [{MIN_WINDOW}, {min(nr, nc)}] for {nr}x{nc}")
    return [Window(r, c, min(size, nr - r), min(size, nc - c))
            for r in range(0, nr, size) for c in range(0, nc, size)]


# ---- description ----------------------------------------------------------------

@dataclass(frozen=True)
class DescriptorConfig:
    beta0: float = 0.0625
    d: int = 4
    l_max: int = 128
    orientation_normalize: bool = True

    def __post_init__(self):
        if self.beta0 <= 0:
            raise ConfigError(f"beta0 must be positive, got {self.beta0}")
        if self.d < 1:
            raise ConfigError(f"subregion grid count must be >= 1, got {self.d}")
        if self.l_max < 1:
            raise ConfigError(f"l_max must be >= 1, got {self.l_max}")

    @property
    def length(self) -> int:
        return self.d * self.d * ORIENTATION_BINS


def region_size(scale: int, cfg) -> int:
    """descriptor.py:82-95 (host arithmetic, same as the library's)."""
    if scale > cfg.l_max:
        raise ConfigError(f"scale {scale} exceeds configured l_max {cfg.l_max}")
    beta = cfg.beta0 * (scale / cfg.l_max) ** -0.5
    w = int(math.floor(beta * scale * cfg.d + 0.5))
    w = min(w, scale)
    w -= w % cfg.d
    return max(w, cfg.d)


@dataclass(eq=False)
class DescribedFeatures:
    image_id: str
    features: list
    descriptors: object  # (n, d*d*8) float64 numpy, or a device tensor


@dataclass(frozen=True, eq=False)
class DescriptorVector:
    values: np.ndarray
    feature: FeaturePoint
    region_size: int
    subregion_size: int


# ---- matching -------------------------------------------------------------------

@dataclass(frozen=True)
class MatcherConfig:
    """matcher.py:16-25, plus ``ratio`` for the extra "ratio_test" strategy."""

    delta_s: float = 0.35
    strategy: str = STRATEGY_NEAREST
    ratio: float = 0.8

    def __post_init__(self):
        if self.delta_s <= 0:
            raise ConfigError(f"delta_s must be positive, got {self.delta_s}")
        if self.strategy not in (STRATEGY_THRESHOLD_ALL, STRATEGY_NEAREST, STRATEGY_RATIO):
            raise ConfigError(f"unknown match strategy {self.strategy!r}")
        if not 0 < self.ratio <= 1:
            raise ConfigError(f"ratio must be in (0, 1], got {self.ratio}")


@dataclass(frozen=True)
class MatchPair:
    p1: tuple
    p2: tuple
    delta: float
    ref1: int
    ref2: int


# ---- registration ---------------------------------------------------------------

@dataclass(frozen=True)
class RigidTransform:
    """Rotation + translation on (x, y) = (col, row); theta kept in (-pi, pi]."""

    theta: float
    t_x: float
    t_y: float

    def __post_init__(self):
        t = math.remainder(self.theta, 2.0 * math.pi)
        if t <= -math.pi:
            t += 2.0 * math.pi
        object.__setattr__(self, "theta", t)

    @classmethod
    def identity(cls) -> "RigidTransform":
        return cls(0.0, 0.0, 0.0)

    @property
    def matrix(self) -> np.ndarray:
        c, s = math.cos(self.theta), math.sin(self.theta)
        return np.array([[c, -s, self.t_x], [s, c, self.t_y], [0.0, 0.0, 1.0]])

    def inverse(self) -> "RigidTransform":
        c, s = math.cos(self.theta), math.sin(self.theta)
        return RigidTransform(-self.theta, -(c * self.t_x + s * self.t_y), -(-s * self.t_x + c * self.t_y))

    def compose(self, inner: "RigidTransform") -> "RigidTransform":
        c, s = math.cos(self.theta), math.sin(self.theta)
        return RigidTransform(self.theta + inner.theta, c * inner.t_x - s * inner.t_y + self.t_x,
                              s * inner.t_x + c * inner.t_y + self.t_y)

    def transform_points(self, points) -> np.ndarray:
        pts = np.asarray(points, dtype=np.float64)
        c, s = math.cos(self.theta), math.sin(self.theta)
        out = np.empty_like(pts)
        out[..., 0] = c * pts[..., 0] - s * pts[..., 1] + self.t_x
        out[..., 1] = s * pts[..., 0] + c * pts[..., 1] + self.t_y
        return out


@dataclass(frozen=True)
class RansacConfig:
    iterations: int = 2000
    inlier_tol: float = 3.0
    min_inliers: int = 8
    seed: int = 0

    def __post_init__(self):
        if self.iterations < 1:
            raise ConfigError("iterations must be >= 1")
        if self.inlier_tol <= 0:
            raise ConfigError("inlier_tol must be positive")
        if self.min_inliers < 2:
            raise ConfigError("min_inliers must be >= 2")


@dataclass(eq=False)
class RegistrationResult:
    transform: RigidTransform
    inliers: list
    residual_rms: float
    consensus_size: int = 0


def apply_transform(transform, point) -> tuple:
    x, y = point
    c, s = math.cos(transform.theta), math.sin(transform.theta)
    return (c * x - s * y + transform.t_x, s * x + c * y + transform.t_y)


# ---- reference interop ---------------------------------------------------------

def reference_module(name: str, *objs):
    """``peakstitch.<name>`` when any of ``objs`` is an object of the reference
    package (its dataclasses), else None.  The drop-ins then build their
    results from the reference's own classes, so code written against the
    reference (``==`` on ``FeaturePoint``/``MatchPair``, ``isinstance``) sees
    exactly its own types."""
    for o in objs:
        if type(o).__module__.split(".", 1)[0] == "peakstitch":
            import importlib

            return importlib.import_module("peakstitch." + name)
    return None
