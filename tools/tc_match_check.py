"""Diagnostic: tensor-core matcher vs the exact float64 path on the same inputs."""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.records import DescriptorConfig  # noqa: E402


def run(d1, d2, exact):
    if exact:
        os.environ["PS_MATCH_EXACT"] = "1"
    else:
        os.environ.pop("PS_MATCH_EXACT", None)
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = device.match(d1, d2)
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in r], time.perf_counter() - t


def compare(name, d1, d2):
    (e1, e2, ed), te = run(d1, d2, True)
    (g1, g2, gd), tg = run(d1, d2, False)
    (g1, g2, gd), tg = run(d1, d2, False)
    ok = np.array_equal(e1, g1) and np.array_equal(e2, g2) and np.array_equal(ed, gd)
    print(f"{name}: n={d1.shape[0]}x{d2.shape[0]} matches exact={len(e1)} tc={len(g1)} equal={ok} "
          f"t_exact={te*1e3:.1f}ms t_tc={tg*1e3:.1f}ms", flush=True)
    return ok


os.environ["PS_TC_MIN_PAIRS"] = "0"
rng = np.random.default_rng(0)
A = torch.from_numpy(rng.random((1000, 128), dtype=np.float32)).cuda()
A = A / A.norm(dim=1, keepdim=True)
B = torch.from_numpy(rng.random((900, 128), dtype=np.float32)).cuda()
B = B / B.norm(dim=1, keepdim=True)
B[:400] = A[:400] + 0.01 * torch.randn_like(A[:400])
B[500:520] = A[7]
ok = compare("random", A, B)
a, b = scenes.config1_pair(0)
cfg = DescriptorConfig(0.0625, 4, 64, True)
ds = []
for im in (a, b):
    t = torch.from_numpy(im).cuda()
    kp = device.detect(t, (16, 32, 64), meta=False)
    ds.append(device.describe(t, kp, cfg)[0])
ok &= compare("C1", ds[0], ds[1])

if len(sys.argv) > 1 and sys.argv[1] == "c4":
    t0 = time.time()
    a, b = scenes.config4_pair(0)
    print(f"C4 scene {time.time()-t0:.1f}s", flush=True)
    cfg = DescriptorConfig(0.0625, 4, 36, True)
    ds = []
    for im in (a, b):
        t = torch.from_numpy(im).cuda()
        kp = device.detect(t, (36,), meta=False)
        ds.append(device.describe(t, kp, cfg, scale_set=(36,))[0])
    print("C4 keypoints", ds[0].shape[0], ds[1].shape[0], flush=True)
    ok &= compare("C4", ds[0], ds[1])
    for _ in range(3):
        _, tg = run(ds[0], ds[1], False)
        print(f"C4 tc {tg*1e3:.2f} ms  pair-matches/s {ds[0].shape[0]*ds[1].shape[0]/tg:.3e}", flush=True)
    sys.exit(0 if ok else 1)
sys.exit(0 if ok else 1)
