"""One C5 pair's tensor-core match (16,320^2) for ncu launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

cfg = PipelineConfig(window_min=16, window_max=64)
sizes, dcfg = cfg.scale_set().sizes, cfg.descriptor_config()
a, b, _ = scenes.config5_pair(0)
g = device.as_device_images(torch.from_numpy(np.stack([a, b])).cuda(), rgb=True)
kp = device.detect(g, sizes, meta=False)
d = device.describe(g, kp, dcfg, scale_set=kp.scale_set)
for _ in range(2):
    r1, r2, _ = device.match(d[0], d[1])
torch.cuda.synchronize()
print("matches", int(r1.shape[0]))
