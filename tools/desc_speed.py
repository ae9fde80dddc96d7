"""C2 describe time (64 x 1600x2688, L 8..128; the headline's dominant
kernel) with CUDA events; prints ms per batch.  Used for A/B builds:
  for f in abvar/desc_*.so; do cp $f paper_2405_08578_b200/libpeakstitch_b200.so; python tools/desc_speed.py; done"""
import multiprocessing as mp
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.records import DescriptorConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cache = "/tmp/c2_batch_%d.npy" % n
if os.path.exists(cache):
    host = np.load(cache)
else:
    with mp.get_context("fork").Pool(16) as pool:
        host = np.stack(pool.map(scenes._scene_job, [(1600, 2688, k) for k in range(n)]))
    np.save(cache, host)
imgs = torch.from_numpy(host).cuda()
dimg = device.DeviceImages(imgs, "u8", device.default_alpha(1600, 2688))
cfg = DescriptorConfig(0.0625, 4, 128, True)
kp = device.detect(dimg, (8, 16, 32, 64, 128), meta=False)
desc = torch.empty((n, kp.cap, 128), dtype=torch.float32, device="cuda")
for _ in range(3):
    device.describe_into(dimg, kp, cfg, desc, scale_set=kp.scale_set)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    device.describe_into(dimg, kp, cfg, desc, scale_set=kp.scale_set)
e1.record()
torch.cuda.synchronize()
print(f"describe C2 x{n}: {e0.elapsed_time(e1) / 10:.3f} ms")
