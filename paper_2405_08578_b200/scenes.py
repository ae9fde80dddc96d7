"""Seeded synthetic scenes for the five BASELINE configurations.

Benchmark/test infrastructure, not part of the hot path.  The reference
ships no generator for the BASELINE "blurred noise + filled shapes" scenes
(its own ``synthetic.make_texture`` at
reference ``pkg/src/peakstitch/synthetic.py:21-36`` is a different texture),
so the parameters below are pinned here and every generated array is
identified by the SHA-256 of its bytes (``scene_digest``).

Parameters:
  1. white noise U[0, 255) float64 from ``default_rng(seed)``;
  2. separable Gaussian blur, sigma 3, radius 12, mirror ("reflect") borders;
  3. min-max stretch to [0, 255];
  4. ``round(200 * H * W / 2048**2)`` filled shapes painted in order, each a
     rectangle or a disk with probability 1/2: rectangle sides U[8, 256]*s,
     disk radius U[4, 128]*s, s = sqrt(H*W)/2048, centre uniform over the
     image, integer intensity U{0..255};
  5. rint, clip to [0, 255], uint8.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

SIGMA = 3.0
RADIUS = 12
SHAPES_AT_2048 = 200


def _gauss_taps() -> np.ndarray:
    x = np.arange(-RADIUS, RADIUS + 1, dtype=np.float64)
    k = np.exp(-(x * x) / (2.0 * SIGMA * SIGMA))
    return k / k.sum()


def _blur_axis(a: np.ndarray, axis: int) -> np.ndarray:
    # scipy's C correlate1d (half-sample mirror borders); pinned by the digests
    # in tests/golden/scene_digests.json
    from scipy.ndimage import correlate1d

    return correlate1d(a, _gauss_taps(), axis=axis, mode="reflect")


def scene(h: int, w: int, seed: int = 0) -> np.ndarray:
    """(h, w) uint8 noise+shapes scene, deterministic in (h, w, seed)."""
    rng = np.random.default_rng(seed)
    f = rng.uniform(0.0, 255.0, size=(h, w))
    f = _blur_axis(_blur_axis(f, 0), 1)
    lo, hi = float(f.min()), float(f.max())
    f = (f - lo) * (255.0 / (hi - lo))
    s = math.sqrt(h * w) / 2048.0
    n_shapes = int(round(SHAPES_AT_2048 * h * w / 2048.0**2))
    for _ in range(n_shapes):
        kind = rng.integers(0, 2)
        cy = rng.uniform(0, h)
        cx = rng.uniform(0, w)
        val = float(rng.integers(0, 256))
        if kind == 0:
            sh = rng.uniform(8, 256) * s
            sw = rng.uniform(8, 256) * s
            r0, r1 = int(max(0, round(cy - sh / 2))), int(min(h, round(cy + sh / 2)))
            c0, c1 = int(max(0, round(cx - sw / 2))), int(min(w, round(cx + sw / 2)))
            f[r0:r1, c0:c1] = val
        else:
            rad = rng.uniform(4, 128) * s
            r0, r1 = int(max(0, math.floor(cy - rad))), int(min(h, math.ceil(cy + rad) + 1))
            c0, c1 = int(max(0, math.floor(cx - rad))), int(min(w, math.ceil(cx + rad) + 1))
            if r1 <= r0 or c1 <= c0:
                continue
            yy = np.arange(r0, r1, dtype=np.float64)[:, None] - cy
            xx = np.arange(c0, c1, dtype=np.float64)[None, :] - cx
            m = yy * yy + xx * xx <= rad * rad
            f[r0:r1, c0:c1][m] = val
    return np.clip(np.rint(f), 0, 255).astype(np.uint8)


def scene_digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---- per-config inputs -----------------------------

def config1_pair(seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """C1: two 768x1024 crops of scene(2048, 2048), 40% overlap, integer shift."""
    s = scene(2048, 2048, seed)
    return s[640:1408, 0:1024].copy(), s[640:1408, 614:1638].copy()


def _scene_job(args):
    return scene(*args)


def config2_batch(n: int = 64, h: int = 1600, w: int = 2688, seed0: int = 0,
                  workers: int = 0) -> np.ndarray:
    """C2: n independent scenes, image k seeded with seed0 + k; (n, h, w) uint8."""
    out = np.empty((n, h, w), dtype=np.uint8)
    jobs = [(h, w, seed0 + k) for k in range(n)]
    if workers > 1 and n > 1:
        import multiprocessing as mp

        with mp.get_context("fork").Pool(workers) as pool:
            for k, img in enumerate(pool.imap(_scene_job, jobs)):
                out[k] = img
    else:
        for k, job in enumerate(jobs):
            out[k] = scene(*job)
    return out


def config4_pair(seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """C4: two 8192x8192 crops of scene(8192, 12288) with 50% overlap."""
    s = scene(8192, 12288, seed)
    return s[:, 0:8192].copy(), s[:, 4096:12288].copy()


def _warp_crop(src: np.ndarray, r0: int, c0: int, h: int, w: int, theta: float, scale: float) -> np.ndarray:
    """Crop [r0:r0+h, c0:c0+w] of src rotated by theta and scaled about its
    centre: output (r, c) samples src at centre + R(theta) (p - centre) / scale,
    bilinear, clamp-to-edge."""
    from scipy.ndimage import map_coordinates

    cy, cx = r0 + (h - 1) / 2.0, c0 + (w - 1) / 2.0
    rr, cc = np.meshgrid(np.arange(h, dtype=np.float64) + r0 - cy, np.arange(w, dtype=np.float64) + c0 - cx,
                         indexing="ij")
    ct, st = math.cos(theta), math.sin(theta)
    sx = (ct * cc - st * rr) / scale + cx
    sy = (st * cc + ct * rr) / scale + cy
    return map_coordinates(src.astype(np.float64), [sy, sx], order=1, mode="nearest")


def config3_images(seed: int = 0, rot_deg: float = 5.0, scale_range=(0.95, 1.05),
                   noise: float = 2.0) -> tuple[list, list]:
    """C3: 3x3 grid of 1600x2688 crops of scene(4200, 7000).

    Each crop gets rotation U[-5, 5] deg and scale U[0.95, 1.05] about its
    centre (bilinear, clamp-to-edge), + N(0, 2^2) noise, rint/clip to uint8;
    the order is shuffled by default_rng(seed).permutation(9).  Returns
    (images, truth) with truth[k] = (row0, col0, theta, scale) of image k.
    """
    src = scene(4200, 7000, seed)
    rng = np.random.default_rng(seed + 1000)
    h, w = 1600, 2688
    out, truth = [], []
    for r0 in (180, 1300, 2420):
        for c0 in (274, 2156, 4037):
            theta = math.radians(rng.uniform(-rot_deg, rot_deg))  # the defaults are the config; other
            sc = rng.uniform(*scale_range)  # values (diagnostics) consume the same draws
            img = _warp_crop(src, r0, c0, h, w, theta, sc) + rng.normal(0.0, noise, size=(h, w))
            out.append(np.clip(np.rint(img), 0, 255).astype(np.uint8))
            truth.append((r0, c0, theta, sc))
    order = np.random.default_rng(seed).permutation(9)
    return [out[k] for k in order], [truth[k] for k in order]


LUMA = np.array([0.299, 0.587, 0.114])  # BT.601 weights (reference imaging.py:21)


def gray_bt601(rgb: np.ndarray) -> np.ndarray:
    """The reference's to_grayscale (imaging.py:66-68): float64 rgb @ weights."""
    return np.asarray(rgb, dtype=np.float64) @ LUMA


def _homography_warp(img: np.ndarray, H: np.ndarray) -> np.ndarray:
    """Output (r, c) samples img at H^-1 (c, r, 1), bilinear, clamp-to-edge."""
    from scipy.ndimage import map_coordinates

    h, w = img.shape[:2]
    Hi = np.linalg.inv(H)
    rr, cc = np.meshgrid(np.arange(h, dtype=np.float64), np.arange(w, dtype=np.float64), indexing="ij")
    den = Hi[2, 0] * cc + Hi[2, 1] * rr + Hi[2, 2]
    sx = (Hi[0, 0] * cc + Hi[0, 1] * rr + Hi[0, 2]) / den
    sy = (Hi[1, 0] * cc + Hi[1, 1] * rr + Hi[1, 2]) / den
    chans = img[..., None] if img.ndim == 2 else img
    out = np.stack([map_coordinates(chans[..., k].astype(np.float64), [sy, sx], order=1, mode="nearest")
                    for k in range(chans.shape[-1])], axis=-1)
    return out if img.ndim == 3 else out[..., 0]


def _c5_job(p: int):
    """Pool worker: the two RGB images of C5 pair p."""
    a, b, _ = config5_pair(p)
    return a, b


def config5_pair(p: int, h: int = 1080, w: int = 1920) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """C5 pair p: RGB image 1 (channel c = scene(h, w, 3p + c)) and image 2 =
    centre-anchored homography warp of it (rotation U[-10, 10] deg, scale
    U[0.92, 1.08], perspective p1, p2 in U[-1e-4, 1e-4]) with gain U[0.7, 1.3],
    offset U[-20, 20] and N(0, 5^2) noise; both uint8 (h, w, 3).  Returns
    (img1, img2, H) with H mapping image-1 (x, y) to image-2 (x, y)."""
    img1 = np.stack([scene(h, w, 3 * p + c) for c in range(3)], axis=-1)
    rng = np.random.default_rng(10_000 + p)
    th = math.radians(rng.uniform(-10.0, 10.0))
    s = rng.uniform(0.92, 1.08)
    p1, p2 = rng.uniform(-1e-4, 1e-4, size=2)
    cx, cy = (w - 1) / 2.0, (h - 1) / 2.0
    T = np.array([[1, 0, -cx], [0, 1, -cy], [0, 0, 1.0]])
    A = np.array([[s * math.cos(th), -s * math.sin(th), 0], [s * math.sin(th), s * math.cos(th), 0], [p1, p2, 1.0]])
    H = np.linalg.inv(T) @ A @ T
    warped = _homography_warp(img1, H)
    gain, off = rng.uniform(0.7, 1.3), rng.uniform(-20.0, 20.0)
    img2 = warped * gain + off + rng.normal(0.0, 5.0, size=warped.shape)
    return img1, np.clip(np.rint(img2), 0, 255).astype(np.uint8), H
