"""Drop-in ``ransac_rigid`` / ``estimate_rigid`` (reference
registration.py:107-203) on the GPU.

The seeded sample stream is numpy's PCG64 stream (the reference's own RNG),
drawn on the host; hypothesis fitting, scoring, selection and the refit run
in the C-ABI library.
"""

from __future__ import annotations

import sys

import numpy as np
import torch

from . import _lib, device
from .errors import DegenerateSampleError, RegistrationError
from .records import (RansacConfig, RegistrationResult, RigidTransform, apply_transform, reference_module)

__all__ = ["ransac_rigid", "estimate_rigid", "transfer_errors", "RansacConfig", "RegistrationResult",
           "RigidTransform", "apply_transform", "ransac_points"]


def _points(pairs):
    src = np.array([[p.p1[1], p.p1[0]] for p in pairs], dtype=np.float64).reshape(-1, 2)
    dst = np.array([[p.p2[1], p.p2[0]] for p in pairs], dtype=np.float64).reshape(-1, 2)
    return src, dst


def ransac_points(src, dst, cfg, _ref=None) -> RegistrationResult:
    """RANSAC on (n, 2) (x, y) point arrays (numpy or device tensors)."""
    n = int(src.shape[0])
    if n < cfg.min_inliers:
        raise RegistrationError(f"only {n} candidate pairs, need at least {cfg.min_inliers}")
    s = src if isinstance(src, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64))
    d = dst if isinstance(dst, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(dst, dtype=np.float64))
    out = device.ransac(s.cuda(), d.cuda(), cfg.iterations, cfg.inlier_tol, cfg.min_inliers, cfg.seed)
    if out.status == _lib.PS_ERR_DEGENERATE:
        raise DegenerateSampleError("source points are coincident")
    if not out.ok:
        raise RegistrationError(f"best consensus {out.consensus} below min_inliers {cfg.min_inliers}")
    ref = _ref or reference_module("registration", cfg)
    res_cls, tr_cls = (ref.RegistrationResult, ref.RigidTransform) if ref else (RegistrationResult, RigidTransform)
    return res_cls(transform=tr_cls(out.theta, out.t_x, out.t_y), inliers=out.inliers.tolist(),
                   residual_rms=out.rms, consensus_size=out.consensus)


def ransac_rigid(pairs, cfg) -> RegistrationResult:
    n = len(pairs)
    if n < cfg.min_inliers:
        raise RegistrationError(f"only {n} candidate pairs, need at least {cfg.min_inliers}")
    src, dst = _points(pairs)
    return ransac_points(src, dst, cfg, reference_module("registration", cfg, pairs[0]))


def estimate_rigid(src, dst) -> RigidTransform:
    src = np.asarray(src, dtype=np.float64)
    dst = np.asarray(dst, dtype=np.float64)
    if src.shape != dst.shape or src.ndim != 2 or src.shape[1] != 2:
        raise DegenerateSampleError("need matching (n, 2) point arrays")
    if src.shape[0] < 2:
        raise DegenerateSampleError("need at least 2 correspondences")
    th, tx, ty, st = device.estimate(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda())
    if st != _lib.PS_OK:
        raise DegenerateSampleError("source points are coincident")
    # array arguments carry no type: follow the reference when it is loaded
    ref = sys.modules.get("peakstitch.registration")
    return (ref.RigidTransform if ref else RigidTransform)(theta=th, t_x=tx, t_y=ty)


def transfer_errors(transform, src, dst) -> np.ndarray:
    """Host helper (not on the hot path): forward-transfer error of each pair."""
    pred = transform.transform_points(src)
    diff = np.asarray(dst, dtype=np.float64) - pred
    return np.hypot(diff[:, 0], diff[:, 1])
