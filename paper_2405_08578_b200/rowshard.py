"""Row-sharded nearest_neighbor matching of one large pair over GPUs
(reference matcher.py:57-95).

Rank r holds rows [offset_r, offset_r + n_r) of A and all of B.  The only
exchange steps are the ones the mutual check needs:

  1. local:  nn12, d12 for my rows of A against all of B;
  2. all-reduce(MAX) of the candidate-column flags (nn12 of rows with
     d12 < delta_s), so every rank agrees on the column set J;
  3. local:  for every column in J, the exact first argmin over MY rows;
  4. all-reduce(MIN) of the float64 distance bits (non-negative doubles
     order like their bit patterns), then all-reduce(MIN) of the global row
     among the ranks that hold that minimum -- together the global first
     argmin nn21 (np.argmin ties go to the lowest index);
  5. local acceptance nn21[nn12[i]] == i and d12 < delta_s, then one
     all-gather of the accepted pairs, sorted by (delta, ref1, ref2).

The one-direction nearest search is pluggable (``nearest_fn``) so the
exchange logic is testable on CPU with gloo; on GPUs it is device.nearest
(tcgen05 candidates + exact float64 certification).
"""

from __future__ import annotations

import torch

INT64_MAX = (1 << 63) - 1


def _dist():
    import torch.distributed as dist

    return dist


def _world(group):
    dist = _dist()
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def match_rows_sharded(desc_a_local: torch.Tensor, row_offset: int, desc_b: torch.Tensor, delta_s: float = 0.35,
                       group=None, nearest_fn=None):
    """Returns (ref1, ref2, delta) of the whole pair (same on every rank)."""
    if nearest_fn is None:
        from .device import nearest as nearest_fn
    dist = _dist()
    rank, world = _world(group)
    dev = desc_b.device
    n2 = int(desc_b.shape[0])

    def allreduce(t, op):
        if world > 1:
            dist.all_reduce(t, op=op, group=group)
        return t

    # 1. my rows against all of B
    nn12, d12 = nearest_fn(desc_a_local, desc_b)
    nn12, d12 = nn12.long(), d12
    # 2. candidate columns
    colflag = torch.zeros(n2, dtype=torch.int32, device=dev)
    cand = d12 < delta_s
    colflag[nn12[cand]] = 1
    allreduce(colflag, dist.ReduceOp.MAX)
    J = torch.nonzero(colflag).flatten()
    # 3. the candidate columns against my rows
    if desc_a_local.shape[0] > 0 and J.numel() > 0:
        nn21_l, d21_l = nearest_fn(desc_b[J], desc_a_local)
        bits = d21_l.view(torch.int64).clone()
        grow = nn21_l.long() + row_offset
    else:
        bits = torch.full((J.numel(),), INT64_MAX, dtype=torch.int64, device=dev)
        grow = torch.full((J.numel(),), INT64_MAX, dtype=torch.int64, device=dev)
    # 4. global first argmin per column
    best = allreduce(bits.clone(), dist.ReduceOp.MIN)
    rows = torch.where(bits == best, grow, torch.full_like(grow, INT64_MAX))
    nn21 = allreduce(rows, dist.ReduceOp.MIN)
    # 5. acceptance on my rows, then gather
    colpos = torch.full((n2,), -1, dtype=torch.int64, device=dev)
    colpos[J] = torch.arange(J.numel(), device=dev)
    my_rows = torch.arange(desc_a_local.shape[0], device=dev) + row_offset
    ok = cand.clone()
    ok[cand] = nn21[colpos[nn12[cand]]] == my_rows[cand]
    acc = torch.stack([my_rows[ok].double(), nn12[ok].double(), d12[ok]], dim=1)
    if world > 1:
        cnt = torch.tensor([acc.shape[0]], dtype=torch.int64, device=dev)
        cnts = [torch.zeros_like(cnt) for _ in range(world)]
        dist.all_gather(cnts, cnt, group=group)
        m = int(max(int(c) for c in cnts))
        pad = torch.zeros((m, 3), dtype=torch.float64, device=dev)
        pad[: acc.shape[0]] = acc
        outs = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(outs, pad, group=group)
        acc = torch.cat([o[: int(c)] for o, c in zip(outs, cnts)])
    ref1, ref2, delta = acc[:, 0].long(), acc[:, 1].long(), acc[:, 2]
    # order by (delta, ref1, ref2): stable sorts, least significant key first
    o = torch.argsort(ref1, stable=True)
    o = o[torch.argsort(delta[o], stable=True)]
    return ref1[o], ref2[o], delta[o]
