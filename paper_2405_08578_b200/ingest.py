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
Once per device the table is compared on the GPU with the two-FMA formula
the x86-64 OpenBLAS dgemv kernel evaluates; when all 2^24 entries agree (they
do on this image's hosts) the kernels compute the grey instead of gathering
it from the 128 MB table.
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


def _cuda_device(device):
    dev = torch.device(device if device is not None else "cuda")
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def gray_lut(device=None) -> torch.Tensor:
    """The grey table on ``device`` (cached per device)."""
    dev = _cuda_device(device)
    with _lock:
        t = _dev_luts.get(dev)
    if t is None:
        t = torch.from_numpy(host_gray_lut()).to(dev)
        with _lock:
            _dev_luts[dev] = t
    return t


_formula_ok: dict = {}


def gray_source(device=None):
    """What the RGB8 kernels read the grey from: None when the fused formula
    fma(B, .114, fma(R, .299, G * .587)) reproduces this host's table on all
    2^24 triples (checked once per device with ps_gray_table_check), else
    the table itself."""
    import ctypes as C

    from . import _lib

    dev = _cuda_device(device)
    with _lock:
        ok = _formula_ok.get(dev)
    if ok is None:
        lut = gray_lut(dev)
        bad = torch.zeros(1, dtype=torch.int64, device=dev)
        with torch.cuda.device(dev):
            st = torch.cuda.current_stream().cuda_stream
            _lib.check(_lib.lib().ps_gray_table_check(C.c_void_p(lut.data_ptr()), C.c_void_p(bad.data_ptr()),
                                                      C.c_void_p(st)), "gray_table_check")
        ok = int(bad.item()) == 0
        with _lock:
            _formula_ok[dev] = ok
            if ok:
                _dev_luts.pop(dev, None)  # the formula replaces the 128 MB table
    return None if ok else gray_lut(dev)


def rgb_key(rgb: torch.Tensor) -> torch.Tensor:
    """R<<16 | G<<8 | B of a [..., 3] uint8 tensor (int64)."""
    c = rgb.to(torch.int64)
    return (c[..., 0] << 16) | (c[..., 1] << 8) | c[..., 2]


def to_grayscale_device(rgb: torch.Tensor) -> torch.Tensor:
    """Device twin of the reference's to_grayscale (imaging.py:66-68) for
    uint8 RGB [nr, nc, 3] / [B, nr, nc, 3]: float64 greys with the
    reference's bits (through ps_rgb_to_gray)."""
    import ctypes as C

    from . import _lib
    from .device import as_device_images

    if rgb.dtype != torch.uint8 or rgb.shape[-1] != 3 or rgb.dim() not in (3, 4):
        raise ValueError("expected uint8 [nr, nc, 3] or [B, nr, nc, 3] RGB")
    im = as_device_images(rgb, rgb=True)
    out = torch.empty(im.data.shape[:3], dtype=torch.float64, device=im.data.device)
    _lib.check(_lib.lib().ps_rgb_to_gray(C.byref(im.c_struct()), C.c_void_p(out.data_ptr()),
                                         C.c_void_p(torch.cuda.current_stream().cuda_stream)), "rgb_to_gray")
    return out if rgb.dim() == 4 else out[0]
