"""Batched pair matching (ps_match_batch_async) vs per-pair launches: C3
pair-phase graph replay (CUDA events) and C5 pairs/s through bench.py."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_08578_b200 import mosaic, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

images, _ = scenes.config3_images(0)
images = [torch.from_numpy(np.ascontiguousarray(im)).pin_memory() for im in images]
cfg = PipelineConfig()
for batched in (False, True, False, True):
    mosaic.GpuEngine.batch_match = batched
    eng = mosaic.GraphEngine(cfg)
    for _ in range(2):
        mosaic.build_pairwise_table(images, cfg, engine=eng)
    torch.cuda.synchronize()
    (pg,) = eng._pair_graphs.values()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pg[0].replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        pg[0].replay()
    e1.record()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        mosaic.build_pairwise_table(images, cfg, engine=eng)
        t1.record()
        torch.cuda.synchronize()
        ts.append(t0.elapsed_time(t1))
    print(f"C3 batch_match={batched}: pair graph {e0.elapsed_time(e1) / 20:.3f} ms, table median {np.median(ts):.3f} ms",
          flush=True)
args = argparse.Namespace(no_cpu=True, no_e2e=True)
for batched in (False, True):
    mosaic.GpuEngine.batch_match = batched
    r = bench.bench_c5_pairs(args, 1, 0, torch.device("cuda", 0), n_pairs=256, steps=3, with_cpu=False)
    print(f"C5 batch_match={batched}: {r['value']} pairs/s  batched_eager {r.get('batched_eager_value')}  "
          f"registered {r.get('registered')}", flush=True)
