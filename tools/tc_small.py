"""Diagnostic: one tensor-core nearest() with few Y tiles (fixed-cost probe)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
X = torch.rand((8448, 128), device="cuda", generator=g)
X = X / X.norm(dim=1, keepdim=True)
Y = torch.rand((int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 128), device="cuda", generator=g)
Y = Y / Y.norm(dim=1, keepdim=True)
for _ in range(3):
    device.nearest(X, Y)
torch.cuda.synchronize()
