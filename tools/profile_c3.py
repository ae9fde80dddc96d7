"""C3 pairwise table: per-stage wall times (synchronised) of the batched
engine, and the whole table per engine mode / stream count."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, mosaic, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig, pair_seed  # noqa: E402

images, _ = scenes.config3_images(0)
cfg = PipelineConfig(window_min=32, window_max=128, ransac_iters=2000, ransac_tol=3.0)
for kw in (dict(batched=False), dict(n_streams=1), dict(n_streams=4), dict(graph=1, n_streams=1),
           dict(graph=1, n_streams=4), dict(graph=1, n_streams=8)):
    eng = mosaic.GraphEngine(cfg, n_streams=kw["n_streams"]) if kw.get("graph") else mosaic.GpuEngine(cfg, **kw)
    mosaic.build_pairwise_table(images, cfg, engine=eng)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        mosaic.build_pairwise_table(images, cfg, engine=eng)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"{kw} table {min(ts) * 1e3:.2f} ms (median {sorted(ts)[2] * 1e3:.2f})")

eng = mosaic.GpuEngine(cfg)
acc = {}


def st(name, fn, rep):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    if rep > 0:
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t
    return r


for rep in range(6):
    batch = st("host stack", lambda: torch.stack([torch.from_numpy(np.ascontiguousarray(im)) for im in images]), rep)
    dbatch = st("upload", lambda: batch.to(eng.device), rep)
    kp = st("detect", lambda: device.detect(dbatch, cfg.scale_set().sizes, meta=False), rep)
    desc = st("describe", lambda: device.describe(dbatch, kp, cfg.descriptor_config(), scale_set=kp.scale_set), rep)
    cnt = kp.count.cpu().numpy()
    jobs = [(a, b) for a in range(9) for b in range(a + 1, 9)]
    ms = st("match_many", lambda: device.match_many([(desc[a][: cnt[a]], desc[b][: cnt[b]]) for a, b in jobs],
                                                     0.35, streams=eng._streams()), rep)

    def rans():
        rj = []
        for (a, b), (r1, r2, _) in zip(jobs, ms):
            if int(r1.shape[0]) >= 8:
                s, d = device.pair_points(r1, r2, kp.row[a], kp.col[a], kp.row[b], kp.col[b])
                rj.append((s, d, 2000, 3.0, 8, pair_seed(cfg.seed, a, b)))
        return device.ransac_many(rj, streams=eng._streams())

    st("ransac_many", rans, rep)
print({k: round(v / 5 * 1e3, 3) for k, v in acc.items()}, "ms; matches/pair",
      float(np.mean([int(m[0].shape[0]) for m in ms])))
