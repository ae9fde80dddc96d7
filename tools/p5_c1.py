"""P5 end-to-end check at C1 scale: GPU chain (u8 fast path and float64
path) against the oracle chain (reference bits) on the C1 pair."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import lpsift_oracle as O  # noqa: E402
from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.records import DescriptorConfig  # noqa: E402

a, b = scenes.config1_pair(0)
cfg = DescriptorConfig(0.0625, 4, 64, True)
t0 = time.time()
ref = []
for im in (a, b):
    P = O.ramp(im.astype(np.float64), O.default_alpha(*im.shape))
    kp = O.detect(P, (16, 32, 64))
    ref.append((kp, O.describe(P, kp, 0.0625, 4, 64, True)))
print(f"oracle describe {time.time()-t0:.1f}s", flush=True)
R32 = [r[1].astype(np.float32).astype(np.float64) for r in ref]
w1, w2, wd = O.match(R32[0], R32[1])
print("oracle: distinct rows", len(np.unique(R32[0], axis=0)), "matches", len(w1), flush=True)
for kind in ("u8", "f64raw"):
    ds = []
    for im in (a, b):
        t = torch.from_numpy(im if kind == "u8" else im.astype(np.float64)).cuda()
        kp = device.detect(t, (16, 32, 64), meta=False)
        ds.append(device.describe(t, kp, cfg)[0])
    G = [d.double().cpu().numpy() for d in ds]
    rel = np.max(np.abs(G[0] - ref[0][1]), axis=1) / np.maximum(np.linalg.norm(ref[0][1], axis=1), 1e-300)
    same32 = np.mean(np.all(G[0] == R32[0], axis=1))
    r1, r2, dl = device.match(ds[0], ds[1])
    got = set(zip(r1.cpu().numpy().tolist(), r2.cpu().numpy().tolist()))
    want = set(zip(w1.tolist(), w2.tolist()))
    print(f"{kind}: distinct rows {len(np.unique(G[0], axis=0))} rows identical to oracle f32 {same32:.4f} "
          f"max rel {rel.max():.2e} matches {len(got)} sym-diff {len(got ^ want)}", flush=True)
