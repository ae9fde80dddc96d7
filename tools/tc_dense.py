"""Diagnostic: tensor-core matcher on 100k x 100k random (all-distinct) descriptors."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 103968
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand((n, 128), device="cuda", generator=g)
A = A / A.norm(dim=1, keepdim=True)
B = torch.rand((n, 128), device="cuda", generator=g)
B[: n // 2] = A[: n // 2] + 0.01 * torch.randn((n // 2, 128), device="cuda", generator=g)
B = B / B.norm(dim=1, keepdim=True)
for _ in range(2):
    r = device.match(A, B)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t = time.perf_counter()
    r = device.match(A, B)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t)
t = sorted(ts)[2]
st = device.match_stats()
print(f"n={n} matches={r[0].shape[0]} time={t*1e3:.2f} ms pair-matches/s={n*n/t:.3e} "
      f"algorithmic TFLOP/s={2*n*n*128/t/1e12:.1f} executed MMA TFLOP/s={st['mma_flops']/t/1e12:.1f} stats={st}")
