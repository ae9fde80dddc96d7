"""Per-stage wall times of the C5 pair path (synchronised after each stage)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

cfg = PipelineConfig(window_min=16, window_max=64)
sizes, dcfg = cfg.scale_set().sizes, cfg.descriptor_config()
pairs = []
for p in range(4):
    a, b, _ = scenes.config5_pair(p)
    pairs.append(device.as_device_images(torch.from_numpy(np.stack([a, b])).cuda(), rgb=True))
acc = {}


def stage(name, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    acc[name] = acc.get(name, 0.0) + time.perf_counter() - t
    return r


for rep in range(3):
    if rep == 1:
        acc.clear()
    for g in pairs:
        kp = stage("detect", lambda: device.detect(g, sizes, meta=False))
        d = stage("describe", lambda: device.describe(g, kp, dcfg, scale_set=kp.scale_set))
        r1, r2, _ = stage("match", lambda: device.match(d[0][: kp.cap], d[1][: kp.cap]))
        src, dst = stage("pair_points", lambda: device.pair_points(r1, r2, kp.row[0], kp.col[0], kp.row[1], kp.col[1]))
        stage("ransac", lambda: device.ransac(src, dst, cfg.ransac_iters, cfg.ransac_tol, cfg.min_inliers, cfg.seed))
n = 2 * len(pairs)
print({k: round(v / n * 1e3, 3) for k, v in acc.items()}, "ms per pair; total", round(sum(acc.values()) / n * 1e3, 3))
