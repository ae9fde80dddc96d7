"""Partitioning of the hot path over the GPUs of one node.

One process per GPU (``torch.distributed``, NCCL on GPUs, gloo in the CPU
tests).  The path shards by independent objects, so the data path has no
collective except where a result must reach every rank:

* C2 (detect + describe batches): every rank runs its own batch of images --
  weak scaling, no collective (``image_slots``);
* C5 (independent image pairs, the reference's per-pair
  ``register_prepared``, pipeline.py:189-209): pair q runs on rank
  q % world and one all-gather of the per-pair result rows gives every rank
  the full list in pair order (``register_pairs_sharded``);
* C3 (pairwise table: images, then pairs) lives in ``mosaic.build_pairwise_table``;
  C4 (rows of one large pair) in ``rowshard.match_rows_sharded``.

Timings are reduced with ``max_over_ranks`` (the job ends with its slowest
rank).  The compute is pluggable (``engine``, the contract of
``mosaic.GpuEngine``) so the orchestration is testable on CPU.
"""

from __future__ import annotations

from typing import Sequence

import torch


def group_info(group=None) -> tuple:
    import torch.distributed as dist

    if group is None and not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def image_slots(rank: int, world: int, per_rank: int) -> list:
    """Global image indices (= generator seeds) of ``rank``'s batch under weak
    scaling: rank r owns r*per_rank .. r*per_rank + per_rank - 1, so rank 0's
    batch is the single-GPU configuration and N ranks process N batches."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return list(range(rank * per_rank, (rank + 1) * per_rank))


def round_robin(n: int, rank: int, world: int) -> list:
    """Items q of 0..n-1 with q % world == rank (the pair / image partition)."""
    return list(range(rank, n, world))


def max_over_ranks(values, group=None, device=None) -> list:
    """Element-wise maximum of a list of floats over the ranks of ``group``."""
    import torch.distributed as dist

    vals = [float(v) for v in values]
    rank, world = group_info(group)
    if world == 1:
        return vals
    t = torch.tensor(vals, dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.cpu().tolist()


def register_pairs_sharded(pairs: Sequence, cfg, *, engine, seeds=None, group=None) -> list:
    """Register independent image pairs [(img_a, img_b), ...] over the ranks:
    pair q on rank q % world (prepare both images, match, RANSAC with seed
    ``seeds[q]``, default ``cfg.seed``), then one all-gather of the result rows.
    Returns [(ok, theta, t_x, t_y, n_inliers), ...] in pair order on every rank."""
    import torch.distributed as dist

    rank, world = group_info(group)
    n = len(pairs)
    seeds = [cfg.seed] * n if seeds is None else list(seeds)
    mine = round_robin(n, rank, world)
    rows = torch.zeros((n, 5), dtype=torch.float64)
    if mine:
        imgs = [im for q in mine for im in pairs[q]]
        r, c, d, cnt = engine.prepare(imgs)
        h = [int(x) for x in cnt.cpu().tolist()]
        items = [(r[2 * k], c[2 * k], d[2 * k], h[2 * k], r[2 * k + 1], c[2 * k + 1], d[2 * k + 1], h[2 * k + 1],
                  seeds[q]) for k, q in enumerate(mine)]
        if getattr(engine, "batched", False) and hasattr(engine, "register_many"):
            outs = engine.register_many(items)
        else:
            outs = [engine.register(*it) for it in items]
        for q, (ok, th, tx, ty, ni) in zip(mine, outs):
            rows[q] = torch.tensor([float(ok), th, tx, ty, float(ni)], dtype=torch.float64)
    if world > 1:
        dev = engine.comm_device()
        t = rows.to(dev)
        out = torch.empty((world * n, 5), dtype=t.dtype, device=dev)
        dist.all_gather_into_tensor(out, t, group=group)
        rows = out.view(world, n, 5).sum(dim=0).cpu()  # each pair was computed by exactly one rank, the others hold zeros
    return [(bool(x[0] > 0.5), float(x[1]), float(x[2]), float(x[3]), int(x[4])) for x in rows.tolist()]
