import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2405_08578_b200 import mosaic, scenes
from paper_2405_08578_b200.pipeline import PipelineConfig
images, _ = scenes.config3_images(0)
images = [torch.from_numpy(np.ascontiguousarray(im)).pin_memory() for im in images]
cfg = PipelineConfig(window_min=32, window_max=128, ransac_iters=2000, ransac_tol=3.0)
eng = mosaic.GraphEngine(cfg)
for _ in range(3): mosaic.build_pairwise_table(images, cfg, engine=eng)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(20): mosaic.build_pairwise_table(images, cfg, engine=eng)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(14)
