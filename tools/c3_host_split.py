import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2405_08578_b200 import mosaic, scenes
from paper_2405_08578_b200.pipeline import PipelineConfig
images, _ = scenes.config3_images(0)
images = [torch.from_numpy(np.ascontiguousarray(im)).pin_memory() for im in images]
cfg = PipelineConfig(window_min=32, window_max=128, ransac_iters=2000, ransac_tol=3.0)
eng = mosaic.GraphEngine(cfg, n_streams=8)
for _ in range(3): mosaic.build_pairwise_table(images, cfg, engine=eng)
torch.cuda.synchronize()
orig_p, orig_r = eng.prepare, eng.register_many
T = {}
def tp(im):
    t = time.perf_counter(); o = orig_p(im); T['prepare_host'] = time.perf_counter() - t; return o
def tr(it):
    t = time.perf_counter(); o = orig_r(it); T['register_many (incl. sync)'] = time.perf_counter() - t; return o
eng.prepare, eng.register_many = tp, tr
for _ in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    mosaic.build_pairwise_table(images, cfg, engine=eng)
    torch.cuda.synchronize(); T['total'] = time.perf_counter() - t0
    print({k: round(v * 1e3, 3) for k, v in T.items()})
