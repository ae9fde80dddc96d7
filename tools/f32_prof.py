"""One C2 describe call per policy (for ncu launch lists / captures)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.records import DescriptorConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
pols = sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto"]
host = np.stack([scenes.scene(1600, 2688, k) for k in range(n)])
imgs = torch.from_numpy(host).cuda()
dimg = device.DeviceImages(imgs, "u8", device.default_alpha(1600, 2688))
cfg = DescriptorConfig(0.0625, 4, 128, True)
kp = device.detect(dimg, (8, 16, 32, 64, 128), meta=False)
out = torch.empty((n, kp.cap, 128), dtype=torch.float32, device="cuda")
for pol in pols:
    device.describe_into(dimg, kp, cfg, out, scale_set=kp.scale_set, policy=pol)
torch.cuda.synchronize()
print("done")
