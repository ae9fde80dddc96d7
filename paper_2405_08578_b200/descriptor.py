"""Drop-in ``describe_features`` / ``compute_descriptor`` (reference
descriptor.py:219-269) on the GPU.

Descriptors come back as float64 numpy rows like the reference's; the
device pipeline (``pipeline.prepare_image``) keeps float32 on the GPU.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device
from .detector import device_images_of
from .records import (DescribedFeatures, DescriptorConfig, DescriptorVector, reference_module, region_size)

__all__ = ["describe_features", "compute_descriptor", "DescriptorConfig", "DescribedFeatures", "region_size"]


def _validate(img, features, cfg) -> None:
    nr, nc = img.nr, img.nc
    for f in features:
        region_size(f.scale, cfg)  # ConfigError when scale > l_max (descriptor.py:89-90)
    if min(nr, nc) - 2 < cfg.d:
        raise ValueError(f"{nr}x{nc} image too small for a {cfg.d}x{cfg.d} subregion grid")
    # features anywhere (even outside the image) are accepted: the region is
    # translated inward like the reference's _fit_region (descriptor.py:118-131)


def describe_tensor(img, features, cfg, out64=True):
    """Device descriptors [n, D] (float64 if out64 else float32) of a feature list."""
    n = len(features)
    dev_img = device_images_of(img)
    dev = dev_img.data.device
    rows = torch.tensor([f.row for f in features], dtype=torch.int32).reshape(1, n).to(dev)
    cols = torch.tensor([f.col for f in features], dtype=torch.int32).reshape(1, n).to(dev)
    scales = torch.tensor([f.scale for f in features], dtype=torch.int32).reshape(1, n).to(dev)
    kp = device.Keypoints(row=rows, col=cols, value=torch.zeros((1, n), dtype=torch.float64, device=dev),
                          count=torch.tensor([n], dtype=torch.int32, device=dev), scale=scales,
                          default_scale=int(features[0].scale),
                          scale_set=tuple(sorted({int(f.scale) for f in features})))
    out = device.describe(dev_img, kp, cfg, out64=out64, out32=not out64)
    return out[0]


def describe_features(img, features, cfg) -> DescribedFeatures:
    features = list(features)
    ref = reference_module("descriptor", img, cfg, *features[:1])
    cls = ref.DescribedFeatures if ref else DescribedFeatures
    if not features:
        return cls(image_id=img.source_id, features=[], descriptors=np.zeros((0, cfg.length)))
    _validate(img, features, cfg)
    mat = describe_tensor(img, features, cfg, out64=True).cpu().numpy()
    return cls(image_id=img.source_id, features=features, descriptors=mat)


def compute_descriptor(img, fp, cfg) -> DescriptorVector:
    _validate(img, [fp], cfg)
    vals = describe_tensor(img, [fp], cfg, out64=True)[0].cpu().numpy()
    w = region_size(fp.scale, cfg)
    cap = min(img.nr, img.nc) - 2
    if w > cap:
        w = cap - cap % cfg.d
    ref = reference_module("descriptor", img, fp, cfg)
    cls = ref.DescriptorVector if ref else DescriptorVector
    return cls(values=vals, feature=fp, region_size=w, subregion_size=w // cfg.d)
