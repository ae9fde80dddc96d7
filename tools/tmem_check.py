"""TMEM read-bandwidth probe and the C4 lines' TMEM rooflines (bench.py's own functions)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
print(json.dumps(bench.tmem_probe(dev)))
d = bench.bench_c4_dense(argparse.Namespace(), 0, dev)
print("dense", d["ms_per_pair"], json.dumps(d["tmem_roofline"]))
c = bench.bench_c4_matching(argparse.Namespace(no_cpu=True), 1, 0, dev, with_cpu=False)
print("c4", c["ms_per_pair"], json.dumps(c["tmem_roofline"]))
