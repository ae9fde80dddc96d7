"""One replay of the C3 pair-phase graph between cudaProfilerStart/Stop, for
`ncu --profile-from-start off --metrics gpu__time_duration.sum` launch lists
(kernel time per pair-phase kernel, serialised)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import mosaic, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

images, _ = scenes.config3_images(0)
cfg = PipelineConfig(window_min=32, window_max=128, ransac_iters=2000, ransac_tol=3.0)
eng = mosaic.GraphEngine(cfg, n_streams=int(os.environ.get("NS", "8")))
for _ in range(2):
    mosaic.build_pairwise_table(images, cfg, engine=eng)
torch.cuda.synchronize()
(pg,) = eng._pair_graphs.values()
(ent,) = eng._prep_graphs.values()
torch.cuda.profiler.start()
for g in ent["graphs"]:
    g.replay()
pg[0].replay()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
