"""One C3 composite (nine crops, feather + bilinear) for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_08578_b200 import compositor as K  # noqa: E402

images, pl = bench.c3_placements()
canvas = K.compute_canvas(pl, {k: v.shape for k, v in images.items()})
dimg = {k: torch.from_numpy(v).cuda() for k, v in images.items()}
for _ in range(3):
    K.warp_and_blend_device(dimg, pl, canvas)
torch.cuda.synchronize()
print("canvas", canvas.height, canvas.width)
