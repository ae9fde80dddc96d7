"""Float32 describe kernel vs the float64 kernels (and sampled oracle rows):
accuracy per keypoint and C2 timing of both policies (CUDA events).
  python tools/f32_check.py [n_images]"""
import multiprocessing as mp
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import lpsift_oracle as O  # noqa: E402  (checker only)
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.records import DescriptorConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
with mp.get_context("fork").Pool(16) as pool:
    host = np.stack(pool.map(scenes._scene_job, [(1600, 2688, k) for k in range(n)]))
imgs = torch.from_numpy(host).cuda()
alpha = device.default_alpha(1600, 2688)
dimg = device.DeviceImages(imgs, "u8", alpha)
cfg = DescriptorConfig(0.0625, 4, 128, True)
kp = device.detect(dimg, (8, 16, 32, 64, 128), meta=False)


def run(policy, out64=False):
    return device.describe(dimg, kp, cfg, scale_set=kp.scale_set, policy=policy, out64=out64)


f32 = run("auto")
p32, p64 = run("precise", out64=True)
torch.cuda.synchronize()
cnt = kp.count.cpu().numpy()
k = int(cnt[0])
ref = p64[:, :k].reshape(-1, 128)
got = f32[:, :k].reshape(-1, 128).double()
nrm = torch.linalg.norm(ref, dim=1).clamp_min(1e-300)
rel = ((got - ref).abs().amax(dim=1) / nrm).cpu().numpy()
l2 = (torch.linalg.norm(got - ref, dim=1)).cpu().numpy()
print(f"f32 vs f64: max rel {rel.max():.3e}  p99 {np.quantile(rel, 0.99):.3e}  median {np.median(rel):.3e}  "
      f"max L2 {l2.max():.3e}  rows bit-equal to rounded f64 {(f32[:, :k] == p32[:, :k]).all(dim=2).float().mean().item():.4f}")
bad = np.argsort(rel)[::-1][:5]
print("worst rows", [(int(i // k), int(i % k), float(rel[i])) for i in bad])
# distinct rows (duplicate structure) on image 0
u32 = torch.unique(f32[0, :k], dim=0).shape[0]
u64 = torch.unique(p32[0, :k], dim=0).shape[0]
print(f"distinct rows img0: f32 kernel {u32}, f64 kernel (rounded) {u64} of {k}")
# oracle sample on image 0
P = O.ramp(host[0].astype(np.float64), alpha)
rows, cols = kp.row[0].cpu().numpy(), kp.col[0].cpu().numpy()
rng = np.random.default_rng(0)
worst = 0.0
for i in rng.choice(k, 300, replace=False):
    want = O.describe_one(P, int(rows[i]), int(cols[i]), 8, 0.0625, 4, 128)
    worst = max(worst, np.max(np.abs(f32[0, i].double().cpu().numpy() - want)) / max(np.linalg.norm(want), 1e-300))
print(f"oracle 300 sampled rows: max rel {worst:.3e}")

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for pol in ("auto", "precise", "auto", "precise"):
    out = torch.empty((n, kp.cap, 128), dtype=torch.float32, device="cuda")
    for _ in range(3):
        device.describe_into(dimg, kp, cfg, out, scale_set=kp.scale_set, policy=pol)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        device.describe_into(dimg, kp, cfg, out, scale_set=kp.scale_set, policy=pol)
    e1.record()
    torch.cuda.synchronize()
    print(f"describe C2 x{n} policy {pol}: {e0.elapsed_time(e1) / 10:.3f} ms")
