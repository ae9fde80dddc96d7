"""Drop-in ``detect_features`` (reference detector.py:154-172) on the GPU.

Accepts this package's or the reference's ``RampedImage``.  A RampedImage
built by ``records.apply_linear_ramp`` carries its raw pixels and alpha, and
the ramp is fused into the kernel (8-bit rasters use the integer-key path);
any other RampedImage is uploaded as its float64 ramped raster.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device
from .records import (MIN_WINDOW, POLARITY_MAX, POLARITY_MIN, FeaturePoint, ScaleSet, Window,
                      partition_windows, reference_module, window_count)

__all__ = ["detect_features", "ScaleSet", "FeaturePoint", "Window", "partition_windows", "window_count",
           "MIN_WINDOW", "POLARITY_MAX", "POLARITY_MIN", "device_images_of"]


def _is_u8_valued(a) -> bool:
    if isinstance(a, torch.Tensor):
        if a.dtype == torch.uint8:
            return True
        if a.dtype.is_floating_point:
            return bool(((a >= 0) & (a <= 255) & (a == torch.round(a))).all())
        return False
    a = np.asarray(a)
    if a.dtype == np.uint8:
        return True
    return bool(np.issubdtype(a.dtype, np.floating) and np.all((a >= 0) & (a <= 255) & (a == np.rint(a))))


def device_images_of(img) -> device.DeviceImages:
    """Upload (or wrap) the raster of a RampedImage for the kernels."""
    raw = getattr(img, "raw", None)
    if raw is not None:
        if _is_u8_valued(raw):
            t = raw if isinstance(raw, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(raw))
            t = t.to(torch.uint8) if t.dtype != torch.uint8 else t
            return device.as_device_images(t, img.alpha)
        return device.as_device_images(np.asarray(raw, dtype=np.float64), img.alpha)
    px = img.pixels
    if isinstance(px, torch.Tensor):
        return device.as_device_images(px.to(torch.float64), img.alpha, ramped=True)
    return device.as_device_images(np.asarray(px, dtype=np.float64), img.alpha, ramped=True)


def features_from_arrays(h: dict, cls=FeaturePoint) -> list:
    pol = (POLARITY_MAX, POLARITY_MIN)
    return [cls(int(r), int(c), int(s), pol[int(p)], int(w), float(v))
            for r, c, s, p, w, v in zip(h["row"], h["col"], h["scale"], h["polarity"], h["window"], h["value"])]


def detect_features(img, scales, dedupe: bool = True) -> list:
    """Window extrema over every scale, deduplicated and sorted (scale, window, polarity)."""
    scales.validate_for(img.nr, img.nc)
    kp = device.detect(device_images_of(img), scales.sizes, dedupe=dedupe, meta=True)
    ref = reference_module("detector", img, scales)
    return features_from_arrays(kp.image(0), ref.FeaturePoint if ref else FeaturePoint)
