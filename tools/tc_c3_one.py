"""One asynchronous C3-sized match (two 8,400-keypoint images) between
cudaProfilerStart/Stop -- for ncu captures of the tensor-core kernels at the
pairwise-table size."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import mosaic, scenes, device  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

images, _ = scenes.config3_images(0)
cfg = PipelineConfig(window_min=32, window_max=128)
eng = mosaic.GpuEngine(cfg)
rows, cols, desc, cnt = eng.prepare(images[:2])
for _ in range(2):
    device.match_async(desc[0], desc[1])
torch.cuda.synchronize()
torch.cuda.profiler.start()
device.match_async(desc[0], desc[1])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
