"""RGB ingest on the device.

The reference turns an RGB file into intensities with a float64 BT.601
matrix product (``to_grayscale``, imaging.py:66-68, called from
``load_image`` :71-93).  Those grey bits come from the host BLAS: no fixed
IEEE / FMA evaluation order reproduces them, so the grey of every
possible (R, G, B) is taken from the run host itself, once per process: one
``rgb_all @ LUMA`` over all 2^24 triples (the very same numpy call the
reference makes, row-independent in BLAS), uploaded as a 128 MB device
table.  With it the RGB8 pixel type of the C-ABI

* detects with the exact integer luma key 299R + 587G + 114B (distinct greys
  differ by >= 0.001, far above the ramp span), and
* fuses the ramp onto the table's grey, so keypoint ``value``s and the
  descriptor's raster are the reference's bits;

and ``to_grayscale_device`` returns the reference's grey image itself.
Uploading RGB moves 3 bytes per pixel instead of the 8 of a float64 grey.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

LUMA = np.array([0.299, 0.587, 0.114])  # imaging.py:21 (BT.601)

_lock = threading.Lock()
_host_lut: np.ndarray | None = None
_dev_luts: dict = {}


def host_gray_lut() -> np.ndarray:
    """float64[2^24]: the reference's grey of (R, G, B) at index R<<16 | G<<8 | B."""
    global _host_lut
    with _lock:
        if _host_lut is None:
            k = np.arange(1 << 24, dtype=np.uint32)
            rgb = np.empty((1 << 24, 3), dtype=np.float64)
            rgb[:, 0] = k >> 16
            rgb[:, 1] = (k >> 8) & 255
            rgb[:, 2] = k & 255
            _host_lut = rgb @ LUMA
        return _host_lut


def gray_lut(device=None) -> torch.Tensor:
    """The grey table on ``device`` (cached per device)."""
    dev = torch.device(device if device is not None else "cuda")
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    with _lock:
        t = _dev_luts.get(dev)
    if t is None:
        t = torch.from_numpy(host_gray_lut()).to(dev)
        with _lock:
            _dev_luts[dev] = t
    return t


def rgb_key(rgb: torch.Tensor) -> torch.Tensor:
    """R<<16 | G<<8 | B of a [..., 3] uint8 tensor (int64)."""
    c = rgb.to(torch.int64)
    return (c[..., 0] << 16) | (c[..., 1] << 8) | c[..., 2]


def to_grayscale_device(rgb: torch.Tensor) -> torch.Tensor:
    """Device twin of the reference's to_grayscale (imaging.py:66-68) for
    uint8 RGB: a float64 [..., nr, nc] tensor with the reference's bits."""
    if rgb.dtype != torch.uint8 or rgb.shape[-1] != 3:
        raise ValueError("expected uint8 [..., 3] RGB")
    if not rgb.is_cuda:
        rgb = rgb.cuda()
    return gray_lut(rgb.device)[rgb_key(rgb)]
