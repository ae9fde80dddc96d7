"""One C4-size (8192^2, L = 36) and one C5 RGB batch detection, for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(1)
t = torch.randint(0, 256, (1, 8192, 8192), dtype=torch.uint8, device="cuda", generator=g)
for _ in range(2):
    device.detect(t, (36,), meta=False)
r = torch.randint(0, 256, (64, 1080, 1920, 3), dtype=torch.uint8, device="cuda", generator=g)
for _ in range(2):
    device.detect(device.as_device_images(r, rgb=True), (16, 32, 64), meta=False)
torch.cuda.synchronize()
