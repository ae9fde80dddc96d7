"""Diagnostic: registered pairs of the C3 nine-image table (GPU engine) as
the generator's perturbations are switched off one by one -- shows which
perturbation the reference's rigid 2-point model cannot absorb."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_08578_b200 import mosaic, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402

cfg = PipelineConfig(window_min=32, window_max=128, ransac_iters=2000, ransac_tol=3.0)
ids = [f"img{k}" for k in range(9)]
for label, kw in [("as specified (rot 5, scale 0.95-1.05, noise 2)", {}),  # noqa: E501
                  ("scale 1 (rot 5, noise 2)", dict(scale_range=(1.0, 1.0))),
                  ("rot 0 (scale 0.95-1.05, noise 2)", dict(rot_deg=0.0)),
                  ("scale 0.99-1.01 (rot 5, noise 2)", dict(scale_range=(0.99, 1.01))),
                  ("rot 0, scale 1 (noise 2)", dict(rot_deg=0.0, scale_range=(1.0, 1.0))),
                  ("rot 0, scale 1, noise 0", dict(rot_deg=0.0, scale_range=(1.0, 1.0), noise=0.0)),
                  ("rot 5, scale 1, noise 0", dict(scale_range=(1.0, 1.0), noise=0.0)),
                  ("rot 5, scale 1, noise 0.5", dict(scale_range=(1.0, 1.0), noise=0.5)),
                  ("as specified, noise 0", dict(noise=0.0))]:
    images, truth = scenes.config3_images(0, **kw)
    table = mosaic.build_pairwise_table(images, cfg)
    plan, placed = mosaic.plan_mosaic(table, ids)
    inl = sorted((e.inlier_count for (a, b), e in table.entries.items() if a < b), reverse=True)
    print(f"{label}: registered pairs {len(inl)} of 36, placed {len(placed)} of 9, inliers {inl[:12]}", flush=True)
