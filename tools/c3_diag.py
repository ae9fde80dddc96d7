"""Diagnostic: per-pair matches / RANSAC consensus on the C3 nine-image set."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, mosaic, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

images, truth = scenes.config3_images(0)
for wmin in (32, 16):
    cfg = PipelineConfig(window_min=wmin, window_max=128 if wmin == 32 else 64)
    eng = mosaic.GpuEngine(cfg)
    rows, cols, desc, cnt = eng.prepare(images)
    print("window", wmin, "keypoints", cnt.tolist(), flush=True)
    for a in range(9):
        for b in range(a + 1, 9):
            (ra, ca, ta, sa), (rb, cb, tb, sb) = truth[a], truth[b]
            if abs(ra - rb) > 1200 or abs(ca - cb) > 2000:
                continue
            r1, r2, dl = device.match(desc[a][: cnt[a]], desc[b][: cnt[b]])
            n = int(r1.shape[0])
            cons = -1
            if n >= 8:
                src, dst = device.pair_points(r1, r2, rows[a], cols[a], rows[b], cols[b])
                out = device.ransac(src, dst, 2000, 3.0, 8, 0)
                cons = out.consensus
            print(f"  pair {a}-{b} grid ({ra},{ca})-({rb},{cb}) dtheta={np.degrees(tb-ta):+.2f} "
                  f"scale {sa:.3f}/{sb:.3f}: matches {n} consensus {cons}", flush=True)
