"""Multi-rank partitions of SURVEY.md §8(e) on CPU (gloo, world size 2),
with the oracle engine of test_mosaic_dist standing in for the GPU kernels:

* C2: weak-scaling image slots (each rank its own batch, no collective) --
  the union over ranks is every image exactly once, and each rank's
  keypoints equal a single-process run on the same images;
* C5: independent pairs round-robin over ranks + one all-gather of the result
  rows == the single-rank list, in pair order;
* the max-over-ranks timing reduction.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_08578_b200 import scenes, shard
from paper_2405_08578_b200.pipeline import PipelineConfig

from test_mosaic_dist import CFG, OracleEngine


def c5_like_pairs():
    """Four independent grey pairs (translation-only crops of different scenes)."""
    out = []
    for k in range(4):
        s = scenes.scene(200, 300, 40 + k)
        out.append((np.ascontiguousarray(s[:, :200]), np.ascontiguousarray(s[:, 90:290])))
    return out


def c2_image(seed):
    return scenes.scene(96, 128, seed)


def test_slot_partitions():
    assert shard.image_slots(0, 1, 64) == list(range(64))
    assert shard.image_slots(3, 8, 64) == list(range(192, 256))
    assert sorted(q for r in range(3) for q in shard.round_robin(10, r, 3)) == list(range(10))
    with pytest.raises(ValueError):
        shard.image_slots(2, 2, 4)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eng = OracleEngine(CFG)
        res = shard.register_pairs_sharded(c5_like_pairs(), CFG, engine=eng, seeds=[11, 12, 13, 14])
        mine = shard.image_slots(rank, world, 2)
        r, c, d, cnt = eng.prepare([c2_image(s) for s in mine])
        mx = shard.max_over_ranks([float(rank), -float(rank)])
        q.put((rank, res, mine, [r.numpy(), c.numpy(), d.numpy()], mx))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_c5_pairs_and_c2_slots():
    eng = OracleEngine(CFG)
    want = shard.register_pairs_sharded(c5_like_pairs(), CFG, engine=eng, seeds=[11, 12, 13, 14])
    assert sum(ok for ok, *_ in want) >= 3  # the overlapping pairs register
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    # drain the queue before joining: a child exits only after its (large) item is consumed
    got = dict((r, (res, mine, arrs, mx)) for r, res, mine, arrs, mx in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    seen = []
    for rank, (res, mine, arrs, mx) in got.items():
        assert res == want, f"rank {rank}: gathered pair results differ"
        assert mx == [1.0, -0.0]
        seen += mine
        single = eng.prepare([c2_image(s) for s in mine])  # same images in one process
        for a, b in zip(arrs, single[:3]):
            assert np.array_equal(a, b.numpy())
    assert sorted(seen) == list(range(4))
