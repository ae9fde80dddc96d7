"""Diagnostic: fast 8-bit describe path vs float64 path on the C4 pair."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.records import DescriptorConfig  # noqa: E402

a, b = scenes.config4_pair(0)
cfg = DescriptorConfig(0.0625, 4, 36, True)
out = {}
for kind in ("u8", "f64raw"):
    ds = []
    for im in (a, b):
        t = torch.from_numpy(im if kind == "u8" else im.astype(np.float64)).cuda()
        kp = device.detect(t, (36,), meta=False)
        ds.append(device.describe(t, kp, cfg, scale_set=(36,))[0])
    r = device.match(ds[0], ds[1])
    print(kind, "matches", int(r[0].shape[0]), "distinct rows", len(torch.unique(ds[0], dim=0)),
          "zero entries", float((ds[0] == 0).float().mean()), flush=True)
    out[kind] = ds
d0, d1 = out["u8"][0].double(), out["f64raw"][0].double()
rel = (d0 - d1).abs().max(dim=1).values / d1.norm(dim=1).clamp_min(1e-300)
print("max rel diff", float(rel.max()), "p99", float(rel.quantile(0.99)), "n > 1e-4", int((rel > 1e-4).sum()))
