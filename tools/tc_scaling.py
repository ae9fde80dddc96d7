"""Diagnostic: nn_topk_tc<0> time vs the number of Y tiles at a fixed row
count (run under ncu with PS_TC_SPLIT=1): fixed cost per CTA vs per tile."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
nx = int(sys.argv[1]) if len(sys.argv) > 1 else 8448
X = torch.rand((nx, 128), device="cuda", generator=g)
X = X / X.norm(dim=1, keepdim=True)
for ny in (1024, 4096, 16384, 65536):
    Y = torch.rand((ny, 128), device="cuda", generator=g)
    Y = Y / Y.norm(dim=1, keepdim=True)
    device.nearest(X, Y)
    torch.cuda.synchronize()
