"""One replay of a C5 pair-phase graph (NP pairs, default 64) between
cudaProfilerStart/Stop, for `ncu --profile-from-start off` launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, mosaic, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

NP = int(os.environ.get("NP", "64"))
cfg = PipelineConfig(window_min=16, window_max=64, ransac_iters=2000, ransac_tol=3.0)
pairs = [scenes.config5_pair(k) for k in range(NP)]
batch = torch.from_numpy(np.stack([im for a, b, _ in pairs for im in (a, b)])).cuda()
g = device.as_device_images(batch, rgb=True)
eng = mosaic.GraphEngine(cfg)
rows, cols, desc, count = eng.prepare_device(g)
n = count.cpu().tolist()
items = [(rows[2 * k], cols[2 * k], desc[2 * k], n[2 * k], rows[2 * k + 1], cols[2 * k + 1], desc[2 * k + 1],
          n[2 * k + 1], 1000 + k) for k in range(NP)]
for _ in range(2):
    eng.register_many(items)
torch.cuda.synchronize()
(pg,) = eng._pair_graphs.values()
torch.cuda.profiler.start()
pg[0].replay()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
