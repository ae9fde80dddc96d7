import time, torch, sys
sys.path.insert(0, '/root/repo')
from paper_2405_08578_b200 import device
A = torch.rand(64, 128, device='cuda'); B = torch.rand(64, 128, device='cuda')
for _ in range(5): device.match(A, B)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200): device.match(A, B)
torch.cuda.synchronize()
print("match 64x64 (CUDA-core path):", (time.perf_counter() - t) / 200 * 1e3, "ms")
src = torch.rand(100, 2, device='cuda', dtype=torch.float64) * 100; dst = src + 1
for _ in range(5): device.ransac(src, dst, 2000, 3.0, 8, 0)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(100): device.ransac(src, dst, 2000, 3.0, 8, 0)
torch.cuda.synchronize()
print("ransac n=100:", (time.perf_counter() - t) / 100 * 1e3, "ms")
import os
os.environ["PS_TC_MIN_PAIRS"] = "0"
A = torch.rand(512, 128, device='cuda'); B = torch.rand(512, 128, device='cuda')
for _ in range(5): device.match(A, B)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(100): device.match(A, B)
torch.cuda.synchronize()
print("match 512x512 (tc path):", (time.perf_counter() - t) / 100 * 1e3, "ms")
