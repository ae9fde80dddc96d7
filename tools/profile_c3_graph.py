"""C3 pairwise table through mosaic.GraphEngine: device time of each graph
replay (CUDA events) and host time of the upload / decode around them."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import mosaic, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

images, _ = scenes.config3_images(0)
cfg = PipelineConfig(window_min=32, window_max=128, ransac_iters=2000, ransac_tol=3.0)
for ns in (4, 8, 16):
    eng = mosaic.GraphEngine(cfg, n_streams=ns)
    for _ in range(2):
        mosaic.build_pairwise_table(images, cfg, engine=eng)
    torch.cuda.synchronize()
    (ent,) = eng._prep_graphs.values()
    (pg,) = eng._pair_graphs.values()
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    acc = np.zeros(3)
    for rep in range(10):
        t0 = time.perf_counter()
        eng._upload([np.asarray(im) for im in images], ent)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ev[0].record(st)
        ent["graph"].replay()
        ev[1].record(st)
        pg[0].replay()
        ev[2].record(st)
        torch.cuda.synchronize()
        acc += [t1 - t0, ev[0].elapsed_time(ev[1]) / 1e3, ev[1].elapsed_time(ev[2]) / 1e3]
    acc /= 10
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        mosaic.build_pairwise_table(images, cfg, engine=eng)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"streams={ns}: upload {acc[0] * 1e3:.3f} ms, prepare graph {acc[1] * 1e3:.3f} ms, "
          f"pair graph {acc[2] * 1e3:.3f} ms; whole table median {sorted(ts)[2] * 1e3:.2f} ms")
