"""Describe throughput for w = 16 (scales 32..128) on 16 C2-size images:
fast kernel vs the general kernel (policy="general")."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.records import DescriptorConfig  # noqa: E402

imgs = torch.from_numpy(np.stack([scenes.scene(1600, 2688, s) for s in range(16)])).cuda()
cfg = DescriptorConfig(0.0625, 4, 128, True)
kp = device.detect(imgs, (32, 64, 128), meta=False)
n = int(kp.count.sum())
for mode in ("auto", "general"):
    for _ in range(2):
        device.describe(imgs, kp, cfg, scale_set=kp.scale_set, policy=mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        device.describe(imgs, kp, cfg, scale_set=kp.scale_set, policy=mode)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{mode}: {ms:.3f} ms for {n} keypoints = {n / ms / 1e3:.1f} Mkp/s")
