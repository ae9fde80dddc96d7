"""Diagnostic: C3 pair (0, 1) through the synchronous, asynchronous and batched matchers."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, mosaic, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

imgs, _ = scenes.config3_images()
eng = mosaic.GpuEngine(PipelineConfig())
rows, cols, desc, count = eng.prepare(imgs)
n = count.cpu().tolist()
A, B = desc[0, : n[0]], desc[1, : n[1]]
s1, s2, sd = device.match(A, B, 0.35, path="tensor")
print("sync", s1.shape[0], device.match_stats())
x1, x2, xd = device.match(A, B, 0.35, path="exact")
print("exact", x1.shape[0])
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
a1, a2, ad = device.match_async(A, B, 0.35, out_count=cnt)[:3]
torch.cuda.synchronize()
k = int(cnt.item())
print("async", k)
r1, r2, dl, c = device.match_batch_async([A, B], [(0, 1)], 0.35)
torch.cuda.synchronize()
kb = int(c[0].item())
print("batch", kb)
S = set(zip(s1.tolist(), s2.tolist()))
Bt = set(zip(r1[0, :kb].tolist(), r2[0, :kb].tolist()))
At = set(zip(a1[:k].tolist(), a2[:k].tolist()))
print("batch - sync", sorted(Bt - S), "sync - batch", sorted(S - Bt))
print("async - sync", sorted(At - S), "sync - async", sorted(S - At))
Ad, Bd = A.double(), B.double()
for (i, j) in sorted(Bt - S):
    dcol = (Ad - Bd[j]).norm(dim=1)
    drow = (Bd - Ad[i]).norm(dim=1)
    print(i, j, "d", float(dcol[i]), "col argmin", int(dcol.argmin()), float(dcol.min()), "row argmin", int(drow.argmin()),
          "cols within 0.35 of row argmin-row:", int(((Bd - Ad[int(dcol.argmin())]).norm(dim=1) < 0.35).sum()))
