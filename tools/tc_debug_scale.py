import os, sys
sys.path.insert(0, '.')
os.environ["PS_TC_MIN_PAIRS"] = "0"
import numpy as np, torch
from paper_2405_08578_b200 import device
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 50.0
rng = np.random.default_rng(int(scale * 1000))
X = (rng.random((260, 128)) * scale).astype(np.float32)
Y = (rng.random((300, 128)) * scale).astype(np.float32)
Y[:100] = X[:100] + np.float32(0.01 * scale) * rng.standard_normal((100, 128)).astype(np.float32)
try:
    idx, d = device.nearest(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda())
    torch.cuda.synchronize()
    print("ok", idx[:5].tolist())
except Exception as e:
    print("ERR", e)
