"""C2 describe timing (64 x 1600x2688) of the given policies, CUDA events."""
import multiprocessing as mp
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.records import DescriptorConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
pols = sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto"]
tag = sys.argv[3] if len(sys.argv) > 3 else ""
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
out = torch.empty((n, kp.cap, 128), dtype=torch.float32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for pol in pols:
    for _ in range(3):
        device.describe_into(dimg, kp, cfg, out, scale_set=kp.scale_set, policy=pol)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        device.describe_into(dimg, kp, cfg, out, scale_set=kp.scale_set, policy=pol)
    e1.record()
    torch.cuda.synchronize()
    print(f"{tag} describe C2 x{n} policy {pol}: {e0.elapsed_time(e1) / 10:.3f} ms")
