"""Profiling driver: one C4 match (tensor-core path) after a warm-up."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.records import DescriptorConfig  # noqa: E402

a, b = scenes.config4_pair(0)
cfg = DescriptorConfig(0.0625, 4, 36, True)
ds = []
for im in (a, b):
    t = torch.from_numpy(im).cuda()
    kp = device.detect(t, (36,), meta=False)
    ds.append(device.describe(t, kp, cfg, scale_set=(36,))[0])
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    r = device.match(ds[0], ds[1])
torch.cuda.synchronize()
import time
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    r = device.match(ds[0], ds[1])
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print("matches", int(r[0].shape[0]), "C4 match ms", round(sorted(ts)[2] * 1e3, 3), device.match_stats())
