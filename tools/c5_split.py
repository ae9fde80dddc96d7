"""C5 phase split: detect + describe of all 512 RGB images (one batched call
each), then the 256 pair matches (match_many), then RANSAC (ransac_many);
wall clock with a synchronize around each phase, median of 3."""
import multiprocessing as mp
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

n_pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = PipelineConfig(window_min=16, window_max=64)
sizes, dcfg = cfg.scale_set().sizes, cfg.descriptor_config()
with mp.get_context("fork").Pool(16) as pool:
    pairs = list(pool.imap(scenes._c5_job, range(n_pairs)))
allimg = device.as_device_images(torch.from_numpy(np.stack([x for ab in pairs for x in ab])).cuda(), rgb=True)
streams = [torch.cuda.Stream() for _ in range(4)]


def phase(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t, r


res = {}
for rep in range(4):
    t_det, kp = phase(lambda: device.detect(allimg, sizes, meta=False))
    t_des, d = phase(lambda: device.describe(allimg, kp, dcfg, scale_set=kp.scale_set))
    t_match, ms = phase(lambda: device.match_many([(d[2 * q], d[2 * q + 1]) for q in range(n_pairs)], cfg.delta_s,
                                                  streams=streams))
    jobs = []
    for q, (r1, r2, _) in enumerate(ms):
        if int(r1.shape[0]) >= cfg.min_inliers:
            src, dst = device.pair_points(r1, r2, kp.row[2 * q], kp.col[2 * q], kp.row[2 * q + 1], kp.col[2 * q + 1])
            jobs.append((src, dst, cfg.ransac_iters, cfg.ransac_tol, cfg.min_inliers, cfg.seed))
    t_ran, _ = phase(lambda: device.ransac_many(jobs, streams=streams))
    if rep:
        for k, v in (("detect", t_det), ("describe", t_des), ("match", t_match), ("ransac", t_ran)):
            res.setdefault(k, []).append(v)
print({k: round(statistics.median(v) * 1e3, 3) for k, v in res.items()}, "ms for", n_pairs, "pairs")
