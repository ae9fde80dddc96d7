"""Pairwise registration table and mosaic planning, sharded over GPUs
(reference mosaic.py:28-180).

``build_pairwise_table`` runs the hot path for every image and every
unordered image pair, exactly as the reference does (same per-pair seeds,
same table convention), but partitions the work over the ranks of a
``torch.distributed`` process group (one process per GPU):

  phase 1  images   k  with k % world == rank  are detected + described;
  exchange one all-gather of the fixed-size keypoint / descriptor slots
           (the only data-path collective: every pair needs both images);
  phase 2  pairs (a, b), a < b, in reference order, are split round-robin;
  gather   one all-gather of the per-pair results (theta, t_x, t_y,
           inliers, ok), after which every rank holds the same table.

The compute is pluggable (``engine``) so the orchestration is testable on
CPU with gloo; the product engine is ``GpuEngine`` (C-ABI kernels).
``plan_mosaic`` is the reference's greedy host planner on the table.
Compositing (warp_and_blend) is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from .errors import ConfigError
from .pipeline import pair_seed
from .records import RigidTransform


# ---- table (mosaic.py:29-55) -------------------------------------------------------

@dataclass(frozen=True)
class PairEntry:
    transform: RigidTransform  # maps the column image's coordinates into the row image's frame
    inlier_count: int


@dataclass(eq=False)
class PairwiseTransformTable:
    n: int
    entries: dict = field(default_factory=dict)

    def present(self, a: int, b: int) -> bool:
        return (a, b) in self.entries

    def get(self, a: int, b: int) -> PairEntry:
        return self.entries[(a, b)]

    def set_pair(self, a: int, b: int, b_to_a: RigidTransform, inliers: int) -> None:
        if a == b:
            raise ValueError("diagonal entries are not allowed")
        self.entries[(a, b)] = PairEntry(b_to_a, inliers)
        self.entries[(b, a)] = PairEntry(b_to_a.inverse(), inliers)

    def neighbor_count(self, a: int, among: set) -> int:
        return sum(1 for b in among if b != a and (a, b) in self.entries)


# ---- engines ----------------------------------------------------------------------------

class GpuEngine:
    """Hot path on the local GPU through the C-ABI (device.py)."""

    batch_match = True  # register_many: every pair's match in one ps_match_batch_async launch sequence

    def __init__(self, cfg, pair_workers: int = 1, batched: bool = True, n_streams: int = 4):
        self.cfg = cfg
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.pair_workers = pair_workers  # concurrent pair registrations (host threads, one stream each)
        self.batched = batched  # register a rank's pairs with register_many (two host syncs in all)
        self.n_streams = n_streams  # streams the batched pairs are spread over

    def comm_device(self):
        return self.device

    def prepare(self, images: list) -> tuple:
        """images -> (rows int32 [B, cap], cols, desc float32 [B, cap, D], count int32 [B]) on device."""
        batch = torch.stack([im if isinstance(im, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(im))
                             for im in images]).to(self.device)
        return self._prepare_dev(batch)

    def _prepare_dev(self, batch) -> tuple:
        """detect + describe a device batch (uint8 [B, nr, nc] tensor or device.DeviceImages, e.g. RGB)."""
        from . import device

        cfg = self.cfg
        nr, nc = (batch.nr, batch.nc) if isinstance(batch, device.DeviceImages) else batch.shape[1:3]
        alpha = cfg.alpha if cfg.alpha is not None else device.default_alpha(nr, nc)
        if isinstance(batch, device.DeviceImages):
            alpha = batch.alpha
        kp = device.detect(batch, cfg.scale_set().sizes, alpha=alpha, meta=False)
        desc = device.describe(batch, kp, cfg.descriptor_config(), alpha=alpha, scale_set=kp.scale_set)
        return kp.row, kp.col, desc, kp.count

    def register_many(self, items):
        """Every pair of ``items`` = [(ra, ca, da, na, rb, cb, db, nb, seed), ...]
        (optionally + (count_a, count_b): device int32 keypoint counts; the
        batched matcher then reads the counts on the device and sizes
        everything by the slots' capacity, so a captured pair graph survives
        frames whose counts differ) with ONE host synchronisation: all matches, point gathers and RANSAC
        runs are enqueued back to back (device.match_many_async, the match
        counts stay on the device and feed ransac_async_dev; pairs spread over
        ``self.streams``), then the result words of every pair are read at once."""
        cfg = self.cfg
        if cfg.matcher_config().strategy != "nearest_neighbor":
            return [self.register(*it) for it in items]
        block, live = self._pairs_dev(items)
        return self._decode(block[:, :8].cpu(), live)

    def _pairs_dev(self, items):
        """Enqueue the whole pair phase; returns (result block [P, W] float64,
        live flags).  No host synchronisation (capturable in a CUDA graph)."""
        from . import device

        cfg = self.cfg
        mc = cfg.matcher_config()
        streams = self._streams()
        counts = torch.zeros(len(items), dtype=torch.int64, device=self.device)
        dev_cnt = all(len(it) > 9 for it in items) and self.batch_match
        if dev_cnt:  # capacity-sized: the device counts decide (registration.py:158-162 on the device)
            caps = [min(int(it[2].shape[0]), int(it[6].shape[0])) for it in items]
        else:
            caps = [min(int(it[3]), int(it[7])) for it in items]
        width = 8 + (max(caps + [8]) + 7) // 8
        block = torch.zeros((len(items), width), dtype=torch.float64, device=self.device)
        rcs = [cfg.ransac_config(it[8]) for it in items]
        live = [caps[q] >= rcs[q].min_inliers for q in range(len(items))]  # registration.py:158-162
        same = len({(rc.iterations, rc.inlier_tol, rc.min_inliers) for rc in rcs}) == 1
        if self.batch_match and same and all(it[2].dim() == 2 and int(it[2].shape[1]) == 128 for it in items):
            # the whole phase as two launch sequences on the current stream:
            # every pair's match (an image's descriptor set -- same rows at the
            # same address -- grouped and tiled once), then every pair's point
            # gather + RANSAC
            sets, index, pairs, set_counts = [], {}, [], []
            for it in items:
                ends = []
                sides = ((it[2], int(it[3]), it[9] if dev_cnt else None),
                         (it[6], int(it[7]), it[10] if dev_cnt else None))
                for d, n, c in sides:
                    if c is not None:
                        n = int(d.shape[0])
                    key = (d.data_ptr(), n, str(d.dtype), c.data_ptr() if c is not None else 0)
                    if key not in index:
                        index[key] = len(sets)
                        sets.append(d[:n])
                        set_counts.append(c)
                    ends.append(index[key])
                pairs.append(tuple(ends))
            r1, r2, _, _ = device.match_batch_async(sets, pairs, mc.delta_s, out_count=counts,
                                                    set_counts=set_counts if dev_cnt else None)
            jobs = [(it[0], it[1], it[4], it[5], caps[q], rcs[q].seed) if live[q] else None
                    for q, it in enumerate(items)]
            rc = rcs[0]
            device.register_batch_async(jobs, r1, r2, counts, rc.iterations, rc.inlier_tol, rc.min_inliers, block)
            return block, live
        outs = device.match_many_async([(it[2][: it[3]], it[6][: it[7]]) for it in items], mc.delta_s, counts,
                                       streams=streams)
        cur = torch.cuda.current_stream(self.device)
        if streams:
            ready = cur.record_event()
            for s in streams:
                s.wait_event(ready)
        for q, (it, (r1, r2, _)) in enumerate(zip(items, outs)):
            rc = rcs[q]
            if not live[q]:
                continue
            s = streams[q % len(streams)] if streams else None
            with torch.cuda.stream(s) if s is not None else _nullcontext():
                src, dst = device.pair_points_dev(r1, r2, counts[q:q + 1], it[0], it[1], it[4], it[5])
                device.ransac_async_dev(src, dst, counts[q:q + 1], caps[q], rc.iterations, rc.inlier_tol,
                                        rc.min_inliers, rc.seed, block[q])
        if streams:
            for s in streams:
                cur.wait_stream(s)
        return block, live

    @staticmethod
    def _decode(h: torch.Tensor, live) -> list:
        from . import _lib

        out = []
        info = h[:, 4:8].contiguous().view(torch.int64)
        for q, ok in enumerate(live):
            if ok and int(info[q, 0]) == _lib.PS_OK:
                out.append((True, float(h[q, 0]), float(h[q, 1]), float(h[q, 2]), int(info[q, 2])))
            else:
                out.append((False, 0.0, 0.0, 0.0, 0))
        return out

    def _streams(self):
        if self.n_streams <= 1:
            return None
        if getattr(self, "_stream_pool", None) is None:
            self._stream_pool = [torch.cuda.Stream(self.device) for _ in range(self.n_streams)]
        return self._stream_pool

    def register(self, ra, ca, da, na, rb, cb, db, nb, seed):
        """match + RANSAC of one pair -> (ok, theta, t_x, t_y, n_inliers)."""
        from . import device
        from .matcher import match_tensors

        cfg = self.cfg
        mc, rc = cfg.matcher_config(), cfg.ransac_config(seed)
        r1, r2, _ = match_tensors(da[:na], db[:nb], mc)
        if int(r1.shape[0]) < rc.min_inliers:
            return (False, 0.0, 0.0, 0.0, 0)
        src, dst = device.pair_points(r1, r2, ra, ca, rb, cb)
        out = device.ransac(src, dst, rc.iterations, rc.inlier_tol, rc.min_inliers, rc.seed)
        if not out.ok:
            return (False, 0.0, 0.0, 0.0, 0)
        return (True, out.theta, out.t_x, out.t_y, int(out.inliers.shape[0]))


class GraphEngine(GpuEngine):
    """GpuEngine for repeated tables of same-shaped image sets (e.g. a camera
    rig stitched frame after frame): each phase is captured once as a CUDA
    graph and then replayed, so the ~40 kernels per pair and the per-image
    detect/describe cost one graph launch per phase instead of ~1,500 host
    launches.  Inputs are re-uploaded (pinned staging) and everything is
    recomputed on every call; a phase is re-captured when its shapes, counts
    or input addresses change."""

    def __init__(self, cfg, n_streams: int = 8):
        super().__init__(cfg, batched=True, n_streams=n_streams)
        self._prep_graphs = {}
        self._pair_graphs = {}
        self.gather_cache = {}  # build_pairwise_table's all-gather outputs, kept at fixed addresses

    prep_chunk = 3  # images per detect/describe graph: chunk k + 1's upload overlaps chunk k's compute

    def prepare(self, images: list) -> tuple:
        """Upload (pinned) and detect + describe, pipelined in chunks of
        ``prep_chunk`` images: a copy stream uploads chunk k + 1 while the
        current stream replays chunk k's graph, which also writes its rows
        into fixed combined outputs (the pair graphs key on their addresses)."""
        arrs = [im if isinstance(im, torch.Tensor) else np.asarray(im) for im in images]
        n = len(arrs)
        key = (n, tuple(arrs[0].shape), str(arrs[0].dtype))
        ent = self._prep_graphs.get(key)
        cur = torch.cuda.current_stream(self.device)
        if ent is None:
            dt = arrs[0].dtype if isinstance(arrs[0], torch.Tensor) else torch.from_numpy(arrs[0][:1]).dtype
            pinned = torch.empty((n,) + tuple(arrs[0].shape), dtype=dt, pin_memory=True)
            static = torch.empty(pinned.shape, dtype=pinned.dtype, device=self.device)
            chunks = [(k, min(k + self.prep_chunk, n)) for k in range(0, n, self.prep_chunk)]
            ent = {"pinned": pinned, "static": static, "chunks": chunks, "graphs": None, "done": None,
                   "copy": torch.cuda.Stream(self.device)}
            self._bound_cache(self._prep_graphs)
            self._prep_graphs[key] = ent
        chunks, static, copy = ent["chunks"], ent["static"], ent["copy"]
        caller_pinned = all(isinstance(a, torch.Tensor) and a.is_pinned() for a in arrs)
        if not caller_pinned and ent["done"] is not None:
            ent["done"].synchronize()  # the previous copies out of the staging buffer have finished
        copy.wait_stream(cur)  # the previous call's readers of `static` come first
        ready = []
        for k0, k1 in chunks:
            with torch.cuda.stream(copy):
                for k in range(k0, k1):
                    if caller_pinned:
                        static[k].copy_(arrs[k], non_blocking=True)
                    else:
                        pv = ent["pinned"][k].numpy()
                        np.copyto(pv, arrs[k].numpy() if isinstance(arrs[k], torch.Tensor) else arrs[k])
                        static[k].copy_(ent["pinned"][k], non_blocking=True)
                ready.append(copy.record_event())
        ent["done"] = copy.record_event()
        if ent["graphs"] is None:
            cur.wait_stream(copy)
            outs = [self._prepare_dev(static[k0:k1]) for k0, k1 in chunks]  # eager warm-up
            rows0, cols0, desc0, cnt0 = outs[0]
            cap, D = desc0.shape[1], desc0.shape[2]
            comb = (torch.empty((n, cap), dtype=rows0.dtype, device=self.device),
                    torch.empty((n, cap), dtype=cols0.dtype, device=self.device),
                    torch.empty((n, cap, D), dtype=desc0.dtype, device=self.device),
                    torch.empty((n,), dtype=cnt0.dtype, device=self.device))
            torch.cuda.synchronize(self.device)
            graphs = []
            for k0, k1 in chunks:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    part = self._prepare_dev(static[k0:k1])
                    for dst, src in zip(comb, part):
                        dst[k0:k1].copy_(src)
                graphs.append(g)
            ent["graphs"], ent["outs"] = graphs, comb
        for g, ev in zip(ent["graphs"], ready):
            cur.wait_event(ev)
            g.replay()
        return ent["outs"]

    def prepare_device(self, batch) -> tuple:
        """detect + describe of a device-resident batch (uint8 tensor or
        device.DeviceImages) as a replayed CUDA graph; the batch's memory is
        the graph's input (re-captured when its address or shape changes)."""
        from . import device

        data = batch.data if isinstance(batch, device.DeviceImages) else batch
        key = ("dev", data.data_ptr(), tuple(data.shape), str(data.dtype))
        ent = self._prep_graphs.get(key)
        if ent is None:
            self._prepare_dev(batch)  # eager warm-up
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                outs = self._prepare_dev(batch)
            self._bound_cache(self._prep_graphs)
            ent = self._prep_graphs[key] = {"graph": g, "outs": outs}
        ent["graph"].replay()
        return ent["outs"]

    max_graphs = 8  # per phase; each graph keeps its own memory pool alive

    def _bound_cache(self, cache: dict) -> None:
        while len(cache) >= self.max_graphs:  # drop the oldest capture (dicts keep insertion order)
            cache.pop(next(iter(cache)))

    def register_many(self, items):
        if self.cfg.matcher_config().strategy != "nearest_neighbor":
            return [self.register(*it) for it in items]
        if all(len(it) > 9 for it in items):  # device counts: keyed on capacities, not on this frame's counts
            key = tuple((it[0].data_ptr(), it[1].data_ptr(), it[2].data_ptr(), int(it[2].shape[0]),
                         it[9].data_ptr(), it[4].data_ptr(), it[5].data_ptr(), it[6].data_ptr(),
                         int(it[6].shape[0]), it[10].data_ptr(), int(it[8])) for it in items)
        else:
            key = tuple((it[0].data_ptr(), it[1].data_ptr(), it[2].data_ptr(), int(it[3]), it[4].data_ptr(),
                         it[5].data_ptr(), it[6].data_ptr(), int(it[7]), int(it[8])) for it in items)
        ent = self._pair_graphs.get(key)
        if ent is None:
            block, live = self._pairs_dev(items)  # eager warm-up; its results are this call's
            res = self._decode(block[:, :8].cpu(), live)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                gblock, glive = self._pairs_dev(items)
            self._bound_cache(self._pair_graphs)
            self._pair_graphs[key] = (g, gblock, glive)
            return res
        g, block, live = ent
        g.replay()
        return self._decode(block[:, :8].cpu(), live)


class _nullcontext:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


# ---- distributed table -------------------------------------------------------------------

def _group_info(group):
    import torch.distributed as dist

    if group is None and not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _all_gather(t: torch.Tensor, world: int, group, cache: dict | None = None, tag: str = "") -> torch.Tensor:
    """All-gather of equal-shaped slots -> [world, ...].  With ``cache`` the
    output buffer is kept per (tag, shape, dtype) so its address is stable
    across calls (graph-replaying engines key their graphs on it)."""
    import torch.distributed as dist

    if world == 1:
        return t.unsqueeze(0)
    shape = (world * t.shape[0],) + tuple(t.shape[1:])
    key = (tag, shape, t.dtype)
    out = cache.get(key) if cache is not None else None
    if out is None:
        out = torch.empty(shape, dtype=t.dtype, device=t.device)
        if cache is not None:
            cache[key] = out
    dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    return out.view((world,) + tuple(t.shape))


def _prepare_groups(engine, imgs):
    """engine.prepare over images of possibly different sizes: one call per
    size (each a batched launch), slots padded to the group's largest
    capacity and returned in the input order."""
    keys = [tuple(im.shape) for im in imgs]
    if len(set(keys)) == 1:
        return engine.prepare(imgs)
    outs, where = [], []
    for key in dict.fromkeys(keys):
        idx = [i for i, k in enumerate(keys) if k == key]
        outs.append(engine.prepare([imgs[i] for i in idx]))
        where.append(idx)
    cap = max(o[2].shape[1] for o in outs)
    order = np.argsort(np.concatenate(where), kind="stable")
    perm = torch.as_tensor(order, device=outs[0][0].device)
    return tuple(torch.cat([_pad_cap(o[f], cap) if f < 3 else o[f] for o in outs])[perm] for f in range(4))


def _pad_cap(t: torch.Tensor, cap: int) -> torch.Tensor:
    """Zero-pad the keypoint axis (dim 1) of a slot tensor to ``cap``."""
    if t.shape[1] >= cap:
        return t
    extra = torch.zeros((t.shape[0], cap - t.shape[1]) + tuple(t.shape[2:]), dtype=t.dtype, device=t.device)
    return torch.cat([t, extra], dim=1)


def _plan_cap(engine, shape) -> int:
    """Keypoint slots per image of this size (the detect plan's count-law bound)."""
    from .pipeline import alloc_plan_cap

    return int(getattr(engine, "plan_cap", lambda nr, nc: alloc_plan_cap(nr, nc, engine.cfg))(shape[0], shape[1]))


def build_pairwise_table(images: Sequence, cfg, *, engine=None, group=None) -> PairwiseTransformTable:
    """mosaic.py:79-112 over the ranks of ``group`` (see module docstring)."""
    n = len(images)
    if n < 2:
        raise ConfigError("pairwise table needs at least 2 images")
    engine = engine or GpuEngine(cfg)
    rank, world = _group_info(group)
    dev = engine.comm_device()
    mixed = len({tuple(im.shape) for im in images}) > 1  # images of different sizes (reference allows them)

    # phase 1: my images (k % world == rank); slots padded to `per` images per rank
    mine = list(range(rank, n, world))
    per = -(-n // world)
    rows, cols, desc, cnt = _prepare_groups(engine, [images[k] for k in mine]) if mine else (None,) * 4
    if rows is None:  # ranks without images contribute empty slots of the agreed shape
        probe = engine.prepare([images[0]])
        rows, cols, desc, cnt = (x[:0] for x in probe)
    if mixed:  # every rank pads its slots to the largest keypoint capacity of any image
        cap = max(_plan_cap(engine, tuple(im.shape)) for im in images)
        rows, cols, desc = (_pad_cap(t, cap) for t in (rows, cols, desc))
    cap, D = desc.shape[1], desc.shape[2]

    def pad(t, fill=0):
        if t.shape[0] == per:
            return t
        extra = torch.full((per - t.shape[0],) + tuple(t.shape[1:]), fill, dtype=t.dtype, device=t.device)
        return torch.cat([t, extra])

    # exchange: every rank receives every image's slots (image k = slot k // world ... see order below)
    gcache = getattr(engine, "gather_cache", None)  # stable gather buffers (GraphEngine)
    g_rows = _all_gather(pad(rows).to(dev), world, group, gcache, "rows")
    g_cols = _all_gather(pad(cols).to(dev), world, group, gcache, "cols")
    g_desc = _all_gather(pad(desc).to(dev), world, group, gcache, "desc")
    g_cnt = _all_gather(pad(cnt).to(dev), world, group, gcache, "cnt")

    h_cnt = g_cnt.cpu().numpy()  # one read of every image's keypoint count

    views = {}  # per-image slot views, built once (tensor indexing costs microseconds per call)

    def img(k):  # image k lives on rank k % world, slot k // world
        if k not in views:
            r, s = k % world, k // world
            views[k] = (g_rows[r, s], g_cols[r, s], g_desc[r, s], int(h_cnt[r, s]))
        return views[k]

    # phase 2: pairs in reference order, round-robin over ranks; on a GPU the
    # rank's pairs run concurrently on a few streams (each pair's small
    # kernels and count read-backs overlap the others')
    jobs = [(a, b) for a in range(n) for b in range(a + 1, n)]
    res = torch.zeros((len(jobs), 5), dtype=torch.float64, device=dev) if world > 1 else None
    mine_q = list(range(rank, len(jobs), world))

    def run(q):
        a, b = jobs[q]
        ra, ca, da, na = img(a)
        rb, cb, db, nb = img(b)
        return engine.register(ra, ca, da, na, rb, cb, db, nb, pair_seed(cfg.seed, a, b))

    workers = getattr(engine, "pair_workers", 1)
    if getattr(engine, "batched", False) and hasattr(engine, "register_many"):
        # the device keypoint counts ride along (int32 slots): the batched
        # matcher reads them on the device, so replayed pair graphs do not
        # depend on this call's counts
        dev_cnt = g_cnt.dtype == torch.int32 and getattr(engine, "batch_match", False)

        def cnt(k):
            return (g_cnt[k % world, k // world].reshape(1),) if dev_cnt else ()

        items = []
        for q in mine_q:
            a, b = jobs[q]
            items.append(img(a) + img(b) + (pair_seed(cfg.seed, a, b),) + (cnt(a) + cnt(b) if dev_cnt else ()))
        outs = engine.register_many(items)
    elif workers > 1 and len(mine_q) > 1:
        import threading
        from concurrent.futures import ThreadPoolExecutor

        local = threading.local()
        torch.cuda.current_stream(dev).synchronize()  # gathered slots ready before other streams read them

        def run_on_stream(q):
            if not hasattr(local, "stream"):
                local.stream = torch.cuda.Stream(dev)
            with torch.cuda.stream(local.stream):
                out = run(q)
            local.stream.synchronize()
            return out

        with ThreadPoolExecutor(max_workers=workers) as ex:
            outs = list(ex.map(run_on_stream, mine_q))
    else:
        outs = [run(q) for q in mine_q]
    rows_h = np.array([[float(ok), th, tx, ty, float(ni)] for ok, th, tx, ty, ni in outs],
                      dtype=np.float64).reshape(-1, 5)
    if world == 1:  # every pair is local: no device round trip
        allres = np.zeros((len(jobs), 5))
        allres[mine_q] = rows_h
    else:
        if mine_q:  # one host-to-device copy of this rank's rows
            res[mine_q] = torch.from_numpy(rows_h).to(dev)
        # gather: each pair was computed by exactly one rank, the others hold zeros
        allres = _all_gather(res, world, group).sum(dim=0).cpu().numpy()
    table = PairwiseTransformTable(n=n)
    for q, (a, b) in enumerate(jobs):
        ok, th, tx, ty, ni = allres[q]
        if ok > 0.5:
            # ransac gives a -> b; the (a, b) entry maps b into a's frame (mosaic.py:108-111)
            table.set_pair(a, b, RigidTransform(th, tx, ty).inverse(), int(ni))
    return table


# ---- planning (reference mosaic.py:113-180, restated on an inlier matrix) ----------------
#
# The reference walks Python sets and re-scans the table per query.  Here the
# table is turned once into an (n, n) matrix of inlier counts (-1 = no
# verified pair) and every query is a vector operation on it; the greedy
# order and both tie rules are the reference's:
#   anchor = free image with the most verified neighbours among the free
#            ones, lowest index on ties (select_reference, :115-119);
#   link   = placed image with the most inliers to the candidate, lowest
#            index on ties (_best_link, :122-127);
#   rounds sweep the free images in index order until a sweep places none
#   (plan_mosaic, :130-180); an anchor with no link into the placed set
#   is dropped to final_unmatched.

@dataclass(eq=False)
class MosaicRound:
    reference_id: str
    stitched_ids: list


@dataclass(eq=False)
class MosaicPlan:
    rounds: list
    final_unmatched: list
    placements: dict = field(default_factory=dict)
    pair_inliers: dict = field(default_factory=dict)
    stage_seconds: dict = field(default_factory=dict)


def inlier_matrix(table: PairwiseTransformTable) -> np.ndarray:
    """(n, n) int64: inlier count of every verified (row, column) entry, -1 elsewhere."""
    W = np.full((table.n, table.n), -1, dtype=np.int64)
    for (a, b), e in table.entries.items():
        W[a, b] = e.inlier_count
    return W


def _anchor(W: np.ndarray, free: np.ndarray) -> int:
    deg = ((W >= 0) & free[None, :]).sum(axis=1)
    idx = np.flatnonzero(free)
    return int(idx[np.argmax(deg[idx])])  # argmax: first (= lowest index) of the maxima


def _link(W: np.ndarray, placed: np.ndarray, c: int):
    score = np.where(placed, W[:, c], -1)
    p = int(np.argmax(score))
    return p if score[p] >= 0 else None


def select_reference(table: PairwiseTransformTable, remaining: set) -> int:
    if not remaining:
        raise ValueError("remaining set is empty")
    free = np.zeros(table.n, dtype=bool)
    free[list(remaining)] = True
    return _anchor(inlier_matrix(table), free)


def plan_mosaic(table: PairwiseTransformTable, ids: Sequence[str]):
    """Greedy rounds over the table -> (MosaicPlan, {image index: placement})."""
    W = inlier_matrix(table)
    free = np.ones(table.n, dtype=bool)
    on_canvas = np.zeros(table.n, dtype=bool)
    pose: dict = {}
    rounds, dropped = [], []

    def attach(c: int, via: int) -> None:
        pose[c] = pose[via].compose(table.get(via, c).transform)
        on_canvas[c], free[c] = True, False

    while free.any():
        a = _anchor(W, free)
        if not on_canvas.any():
            pose[a] = RigidTransform.identity()
            on_canvas[a], free[a] = True, False
        else:
            via = _link(W, on_canvas, a)
            free[a] = False
            if via is None:
                dropped.append(a)
                continue
            attach(a, via)
        joined = []
        swept = True
        while swept:
            swept = False
            for c in np.flatnonzero(free).tolist():  # ascending, re-checked as the canvas grows
                via = _link(W, on_canvas, c)
                if via is not None:
                    attach(c, via)
                    joined.append(c)
                    swept = True
        rounds.append(MosaicRound(ids[a], [ids[i] for i in joined]))
    plan = MosaicPlan(rounds, [ids[i] for i in sorted(dropped)], {ids[i]: t for i, t in pose.items()})
    return plan, pose


def plan_and_stitch(images: Sequence, cfg, *, engine=None, group=None):
    """Reference mosaic.py:183-220 on the GPU -> (plan, composite): the
    pairwise table (sharded over ``group``), the planner above, and the
    device composite of every placed image.  ``images`` are
    IntensityImage-like objects (``pixels``, ``image_id``)."""
    import time

    from . import compositor as K

    if len(images) < 2:
        raise ConfigError("mosaic needs at least 2 images")
    names = [im.image_id for im in images]
    if len(names) != len(set(names)):
        raise ConfigError("image ids must be unique")
    clock = [time.perf_counter()]
    table = build_pairwise_table([im.pixels for im in images], cfg, engine=engine, group=group)
    clock.append(time.perf_counter())
    plan, pose = plan_mosaic(table, names)
    plan.pair_inliers = {(names[a], names[b]): e.inlier_count for (a, b), e in table.entries.items() if a < b}
    clock.append(time.perf_counter())
    order = sorted(pose)
    placements = [K.Placement(names[i], pose[i]) for i in order]
    shapes = {names[i]: tuple(np.asarray(images[i].pixels).shape[:2]) for i in order}
    canvas = K.compute_canvas(placements, shapes)
    composite = K.warp_and_blend({names[i]: images[i].pixels for i in order}, placements, canvas,
                                 blend=cfg.blend, resample=cfg.resample)
    clock.append(time.perf_counter())
    plan.stage_seconds = dict(zip(("pairwise_table", "planning", "compositing"),
                                  (clock[1] - clock[0], clock[2] - clock[1], clock[3] - clock[2])))
    return plan, composite
