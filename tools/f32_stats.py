"""Fallback rates of the float32 describe kernel (build with EXTRA=-DPS_F32_DEBUG)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import _lib, device, scenes  # noqa: E402
from paper_2405_08578_b200.records import DescriptorConfig  # noqa: E402

fn = _lib.lib().ps_f32_debug_counts
buf = (C.c_ulonglong * 8)()
for name, (nr, nc, scales, lmax, seeds) in dict(
        c2=(1600, 2688, (8, 16, 32, 64, 128), 128, range(4)), c1=(768, 1024, (16, 32, 64), 64, range(4)),
        c4=(4096, 4096, (36,), 36, range(1))).items():
    host = np.stack([scenes.scene(nr, nc, s) for s in seeds])
    t = torch.from_numpy(host).cuda()
    kp = device.detect(t, scales, alpha=device.default_alpha(nr, nc), meta=False)
    fn(buf)
    device.describe(t, kp, DescriptorConfig(0.0625, 4, lmax, True), alpha=device.default_alpha(nr, nc),
                    scale_set=kp.scale_set)
    fn(buf)
    n = int(kp.count.sum())
    print(f"{name}: {n} kp, {64 * n} samples/phase: fb8 {buf[0]} ({buf[0] / 64 / n:.2e}/sample), special {buf[1]}, "
          f"exact8 {buf[2]} ({buf[2] / 64 / n:.2e}), fb36 {buf[3]}, exact36 {buf[4]}, lead fails {buf[5]} ({buf[5] / n:.2e}/kp)")
