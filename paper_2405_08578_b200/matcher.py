"""Drop-in ``match_features`` (reference matcher.py:57-95) on the GPU.

float64 descriptor matrices are matched exactly as given (the reference's
float64 arithmetic, bit for bit); float32 device tensors (the pipeline's
descriptors) are upcast exactly.  Output order: (delta, ref1, ref2).
"""

from __future__ import annotations

import numpy as np
import torch

from . import device
from .records import (STRATEGY_NEAREST, STRATEGY_RATIO, STRATEGY_THRESHOLD_ALL, MatcherConfig, MatchPair,
                      reference_module)

__all__ = ["match_features", "MatcherConfig", "MatchPair", "STRATEGY_NEAREST", "STRATEGY_THRESHOLD_ALL", "STRATEGY_RATIO",
           "match_tensors"]


def _dev(desc) -> torch.Tensor:
    if isinstance(desc, torch.Tensor):
        return desc if desc.is_cuda else desc.cuda()
    a = np.asarray(desc)
    if a.dtype != np.float32:
        a = a.astype(np.float64)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def match_tensors(desc1, desc2, cfg):
    """Device (ref1, ref2, delta) of two descriptor matrices."""
    if cfg.strategy == STRATEGY_RATIO:  # extra strategy: the threshold argument carries the ratio
        return device.match(_dev(desc1), _dev(desc2), cfg.ratio, STRATEGY_RATIO)
    return device.match(_dev(desc1), _dev(desc2), cfg.delta_s, cfg.strategy)


def match_features(set1, set2, cfg) -> list:
    n1, n2 = len(set1.features), len(set2.features)
    if n1 == 0 or n2 == 0:
        return []
    r1, r2, dl = match_tensors(set1.descriptors, set2.descriptors, cfg)
    r1, r2, dl = r1.cpu().numpy(), r2.cpu().numpy(), dl.cpu().numpy()
    f1, f2 = set1.features, set2.features
    ref = reference_module("matcher", set1, set2, cfg)
    cls = ref.MatchPair if ref else MatchPair
    return [cls(p1=(f1[i].row, f1[i].col), p2=(f2[j].row, f2[j].col), delta=float(d), ref1=int(i),
                      ref2=int(j)) for i, j, d in zip(r1, r2, dl)]
