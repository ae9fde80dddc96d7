"""Detection throughput of the generic-L kernels (strip kernel) per config:
bytes = c_in * px + 16 B per kept keypoint, CUDA events."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, scenes  # noqa: E402

cases = [("C1 768x1024 L16..64", (1, 768, 1024), (16, 32, 64), False),
         ("C3 9x1600x2688 L32..128", (9, 1600, 2688), (32, 64, 128), False),
         ("C4 8192^2 L36", (1, 8192, 8192), (36,), False),
         ("C4 2x8192^2 L36", (2, 8192, 8192), (36,), False),
         ("C5 64x1080x1920 RGB L16..64", (64, 1080, 1920), (16, 32, 64), True),
         ("C2 64x1600x2688 L8..128", (64, 1600, 2688), (8, 16, 32, 64, 128), False)]
peak = 6534.5
for name, (B, nr, nc), scales, rgb in cases:
    g = torch.Generator(device="cuda").manual_seed(1)
    shape = (B, nr, nc, 3) if rgb else (B, nr, nc)
    t = torch.randint(0, 256, shape, dtype=torch.uint8, device="cuda", generator=g)
    im = device.as_device_images(t, rgb=rgb)
    for _ in range(3):
        kp = device.detect(im, scales, meta=False)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()  # replay: no host launch overhead between the timed launches
    with torch.cuda.graph(gr):
        kp = device.detect(im, scales, meta=False)
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    nbytes = t.numel() + int(kp.count.sum()) * 16
    print(f"{name}: {ms * 1e3:.1f} us, {nbytes / ms / 1e6:.1f} GB/s = {nbytes / ms / 1e6 / peak:.3f} of HBM")
