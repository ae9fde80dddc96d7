"""C3 pairwise table through mosaic.GraphEngine: device time of the prepare
phase (chunked upload + detect/describe graphs) and of the pair-phase graph
replay (CUDA events), and the whole table (pinned host images)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import mosaic, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

images, _ = scenes.config3_images(0)
images = [torch.from_numpy(np.ascontiguousarray(im)).pin_memory() for im in images]
cfg = PipelineConfig(window_min=32, window_max=128, ransac_iters=2000, ransac_tol=3.0)
for chunk in (9, 3, 1):
    eng = mosaic.GraphEngine(cfg)
    eng.prep_chunk = chunk
    for _ in range(2):
        mosaic.build_pairwise_table(images, cfg, engine=eng)
    torch.cuda.synchronize()
    (pg,) = eng._pair_graphs.values()
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    acc = np.zeros(2)
    for rep in range(10):
        torch.cuda.synchronize()
        ev[0].record(st)
        eng.prepare(images)
        ev[1].record(st)
        pg[0].replay()
        ev[2].record(st)
        torch.cuda.synchronize()
        acc += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])]
    acc /= 10
    ts = []
    for _ in range(7):
        t = time.perf_counter()
        mosaic.build_pairwise_table(images, cfg, engine=eng)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"chunk={chunk}: prepare {acc[0]:.3f} ms, pair graph {acc[1]:.3f} ms; "
          f"whole table median {sorted(ts)[3] * 1e3:.2f} ms", flush=True)
