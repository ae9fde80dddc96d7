"""C3 stitch timing vs the number of concurrent pair workers, plus per-stage
wall times of one pair (synchronised)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, mosaic, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

images, _ = scenes.config3_images(0)
cfg = PipelineConfig(window_min=32, window_max=128, ransac_iters=2000, ransac_tol=3.0)
for w in (1, 2, 4, 8):
    eng = mosaic.GpuEngine(cfg, pair_workers=w)
    mosaic.build_pairwise_table(images, cfg, engine=eng)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        mosaic.build_pairwise_table(images, cfg, engine=eng)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"workers={w} table {min(ts) * 1e3:.1f} ms")
eng = mosaic.GpuEngine(cfg)
rows, cols, desc, cnt = eng.prepare(images[:2])
torch.cuda.synchronize()
acc = {}
for rep in range(6):
    def st(name, fn):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        if rep > 0:
            acc[name] = acc.get(name, 0.0) + time.perf_counter() - t
        return r
    t0 = time.perf_counter()
    prep = st("prepare9", lambda: eng.prepare(images))
    r1, r2, _ = st("match", lambda: device.match(desc[0][: int(cnt[0])], desc[1][: int(cnt[1])]))
    if int(r1.shape[0]) >= 8:
        src, dst = st("pair_points", lambda: device.pair_points(r1, r2, rows[0], cols[0], rows[1], cols[1]))
        st("ransac", lambda: device.ransac(src, dst, 2000, 3.0, 8, 0))
print({k: round(v / 5 * 1e3, 3) for k, v in acc.items()}, "ms; matches", int(r1.shape[0]))
