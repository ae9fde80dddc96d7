"""pairs_c5 through bench.py's own function (GraphEngine path), for A/B builds."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else ""
args = argparse.Namespace(no_cpu=True, no_e2e=True)
r = bench.bench_c5_pairs(args, 1, 0, torch.device("cuda", 0), n_pairs=256, steps=3, with_cpu=False)
print(tag, "pairs_c5", r["value"], "pairs/s  batched_eager", r.get("batched_eager_value"))
