"""Compositor on the GPU.

Drop-in for the reference's ``peakstitch.compositor`` (compositor.py:20-160):
``compute_canvas`` sizes the canvas on the host (a handful of corner points,
the reference's own float64 arithmetic), ``warp_and_blend`` resamples every
placed image into it on the device through ``ps_warp_and_blend`` -- one
thread per canvas pixel walking the placements in order, so the feather /
overwrite accumulation and the single-cover passthrough are bit-identical to
the reference.  ``warp_and_blend_device`` is the tensor-in / tensor-out form.

The inverse transform's cos / sin and the per-image canvas blocks are
computed here exactly as the reference computes them (``RigidTransform.inverse``
+ ``transform_points``, registration.py:49-73; snapped corners,
compositor.py:122-129) and handed to the kernel as plain numbers.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _lib
from .records import RigidTransform

BLEND_FEATHER = "feather"
BLEND_OVERWRITE = "overwrite"
RESAMPLE_BILINEAR = "bilinear"
RESAMPLE_NEAREST = "nearest"

_SNAP = 1e-6  # compositor.py:20
_BLEND = {BLEND_FEATHER: _lib.PS_BLEND_FEATHER, BLEND_OVERWRITE: _lib.PS_BLEND_OVERWRITE}
_RESAMPLE = {RESAMPLE_BILINEAR: _lib.PS_RESAMPLE_BILINEAR, RESAMPLE_NEAREST: _lib.PS_RESAMPLE_NEAREST}


@dataclass(frozen=True)
class Placement:
    """An image id plus the transform taking its pixels into the canvas frame."""

    image_id: str
    transform: RigidTransform


@dataclass(eq=False)
class Canvas:
    width: int
    height: int
    origin_offset: tuple[int, int]  # canvas (col, row) + offset = frame (x, y)
    pixels: np.ndarray | None = field(default=None)
    weightmap: np.ndarray | None = field(default=None)


def _frame_corners(transform, nr: int, nc: int) -> np.ndarray:
    """The image's four corners in the canvas frame, snapped to 1e-6 so
    near-identity rotations cannot inflate the bounds (compositor.py:40-41)."""
    pts = transform.transform_points(np.array([[0.0, 0.0], [nc, 0.0], [0.0, nr], [nc, nr]]))
    return np.round(pts / _SNAP) * _SNAP


def compute_canvas(placements: Sequence[Placement], dims: Mapping[str, tuple[int, int]]) -> Canvas:
    """Integer bounding box of every placed image (compositor.py:44-58)."""
    if not placements:
        raise ValueError("need at least one placement")
    pts = np.vstack([_frame_corners(p.transform, *dims[p.image_id]) for p in placements])
    x0, y0 = math.floor(pts[:, 0].min()), math.floor(pts[:, 1].min())
    return Canvas(width=math.ceil(pts[:, 0].max()) - x0, height=math.ceil(pts[:, 1].max()) - y0,
                  origin_offset=(x0, y0))


def _device_pixels(img) -> torch.Tensor:
    """uint8 stays uint8; every other dtype becomes float64 (exact for the
    integer and float32 inputs the reference would promote the same way)."""
    t = img if isinstance(img, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(img))
    if t.dtype != torch.uint8:
        t = t.to(torch.float64)
    return t.to("cuda", non_blocking=False).contiguous()


def _placement_structs(images: Mapping[str, torch.Tensor], placements: Sequence[Placement], canvas: Canvas):
    dx, dy = canvas.origin_offset
    structs = []
    for p in placements:
        px = images[p.image_id]
        nr, nc = int(px.shape[0]), int(px.shape[1])
        corners = _frame_corners(p.transform, nr, nc)
        c_lo = max(math.floor(corners[:, 0].min()) - dx, 0)
        c_hi = min(math.ceil(corners[:, 0].max()) - dx, canvas.width)
        r_lo = max(math.floor(corners[:, 1].min()) - dy, 0)
        r_hi = min(math.ceil(corners[:, 1].max()) - dy, canvas.height)
        if c_lo >= c_hi or r_lo >= r_hi:
            continue  # the image misses the canvas (compositor.py:130-131)
        inv = p.transform.inverse()
        s = _lib.PlacementC()
        s.data = px.data_ptr()
        s.pixel_type = _lib.PS_PIXELS_U8 if px.dtype == torch.uint8 else _lib.PS_PIXELS_F64
        s.nr, s.nc = nr, nc
        s.r_lo, s.r_hi, s.c_lo, s.c_hi = r_lo, r_hi, c_lo, c_hi
        s.row_pitch = int(px.stride(0))
        s.cos_t, s.sin_t = math.cos(inv.theta), math.sin(inv.theta)
        s.t_x, s.t_y = inv.t_x, inv.t_y
        structs.append(s)
    return (_lib.PlacementC * max(len(structs), 1))(*structs), len(structs)


def warp_and_blend_device(images: Mapping[str, torch.Tensor], placements: Sequence[Placement], canvas: Canvas,
                          blend: str = BLEND_FEATHER, resample: str = RESAMPLE_BILINEAR,
                          stream: torch.cuda.Stream | None = None):
    """Device composite: ``images`` are 2-D CUDA tensors (uint8 or float64);
    returns (pixels, weightmap) as float64 CUDA tensors of the canvas shape."""
    if blend not in _BLEND:
        raise ValueError(f"unknown blend mode {blend!r}")
    if resample not in _RESAMPLE:
        raise ValueError(f"unknown resample mode {resample!r}")
    out = torch.empty((canvas.height, canvas.width), dtype=torch.float64, device="cuda")
    wm = torch.empty_like(out)
    arr, n = _placement_structs(images, placements, canvas)
    st = (stream or torch.cuda.current_stream()).cuda_stream
    if n == 0:
        out.zero_()
        wm.zero_()
        return out, wm
    _lib.check(_lib.lib().ps_warp_and_blend(arr, n, canvas.height, canvas.width, int(canvas.origin_offset[0]),
                                            int(canvas.origin_offset[1]), _BLEND[blend], _RESAMPLE[resample],
                                            C.c_void_p(out.data_ptr()), C.c_void_p(wm.data_ptr()),
                                            C.c_void_p(st)), "warp_and_blend")
    return out, wm


def warp_and_blend(images: Mapping[str, np.ndarray], placements: Sequence[Placement], canvas: Canvas,
                   blend: str = BLEND_FEATHER, resample: str = RESAMPLE_BILINEAR) -> np.ndarray:
    """Drop-in for the reference's warp_and_blend (compositor.py:84-160):
    host arrays in, the composite out, ``canvas.pixels`` / ``canvas.weightmap``
    set.  Canvas pixels covered by no image are 0."""
    if blend not in _BLEND:
        raise ValueError(f"unknown blend mode {blend!r}")
    if resample not in _RESAMPLE:
        raise ValueError(f"unknown resample mode {resample!r}")
    used = {p.image_id for p in placements}
    dev = {k: _device_pixels(images[k]) for k in used}
    out, wm = warp_and_blend_device(dev, placements, canvas, blend, resample)
    torch.cuda.current_stream().synchronize()
    canvas.pixels = out.cpu().numpy()
    canvas.weightmap = wm.cpu().numpy()
    return canvas.pixels
