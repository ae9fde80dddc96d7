"""Multi-rank orchestration of the pairwise table (mosaic.build_pairwise_table)
on CPU: world_size 1 vs 2 over gloo, with a CPU engine built from the oracle
(test infrastructure) standing in for the GPU kernels.  Checks the sharding,
the slot all-gather, the per-pair seeds and the table/plan assembly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lpsift_oracle as O
from paper_2405_08578_b200 import mosaic, scenes
from paper_2405_08578_b200.pipeline import PipelineConfig, pair_seed

CFG = PipelineConfig(window_min=16, window_max=32, ransac_iters=300, min_inliers=6)


class OracleEngine:
    """CPU stand-in for GpuEngine (same tensor contract)."""

    def __init__(self, cfg):
        self.cfg = cfg

    def comm_device(self):
        return torch.device("cpu")

    def prepare(self, images):
        cfg = self.cfg
        out_r, out_c, out_d, out_n = [], [], [], []
        for im in images:
            P = O.ramp(im.astype(np.float64), O.default_alpha(*im.shape))
            kp = O.detect(P, cfg.scale_set().sizes)
            d = O.describe(P, kp, cfg.beta0, cfg.d, cfg.window_max, cfg.orientation_normalize)
            out_r.append(torch.from_numpy(kp["row"].astype(np.int32)))
            out_c.append(torch.from_numpy(kp["col"].astype(np.int32)))
            out_d.append(torch.from_numpy(d.astype(np.float32)))
            out_n.append(len(kp))
        return torch.stack(out_r), torch.stack(out_c), torch.stack(out_d), torch.tensor(out_n, dtype=torch.int32)

    def register(self, ra, ca, da, na, rb, cb, db, nb, seed):
        r1, r2, _ = O.match(da[:na].double().numpy(), db[:nb].double().numpy(), self.cfg.delta_s)
        kp1 = {"row": ra.numpy(), "col": ca.numpy()}
        kp2 = {"row": rb.numpy(), "col": cb.numpy()}
        src, dst = O.pair_points(r1, r2, kp1, kp2)
        try:
            r = O.ransac(src, dst, self.cfg.ransac_iters, self.cfg.ransac_tol, self.cfg.min_inliers, seed)
        except O.NoConsensus:
            return (False, 0.0, 0.0, 0.0, 0)
        th, tx, ty = r["model"]
        return (True, th, tx, ty, len(r["inliers"]))


def fragments():
    s = scenes.scene(300, 420, 21)
    crops = [s[r:r + 160, c:c + 224] for r in (0, 140) for c in (0, 98, 196)]
    return [np.ascontiguousarray(c) for c in crops[:5]]


def mixed_fragments():
    """Fragments of different sizes (the reference accepts them, mosaic.py:79-112)."""
    s = scenes.scene(300, 420, 21)
    boxes = [(0, 0, 160, 224), (0, 98, 150, 200), (140, 0, 160, 224), (130, 90, 170, 250), (140, 196, 150, 200)]
    return [np.ascontiguousarray(s[r:r + h, c:c + w]) for r, c, h, w in boxes]


def table_digest(t):
    return sorted((a, b, round(e.transform.theta, 12), round(e.transform.t_x, 9), round(e.transform.t_y, 9),
                   e.inlier_count) for (a, b), e in t.entries.items())


def _worker(rank, world, port, q, mixed=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if mixed:
            q.put((rank, table_digest(mosaic.build_pairwise_table(mixed_fragments(), CFG, engine=OracleEngine(CFG)))))
            return
        t = mosaic.build_pairwise_table(fragments(), CFG, engine=OracleEngine(CFG))
        # an engine with persistent gather buffers (as GraphEngine): two tables through the same buffers
        eng = OracleEngine(CFG)
        eng.gather_cache = {}
        t1 = mosaic.build_pairwise_table(fragments(), CFG, engine=eng)
        t2 = mosaic.build_pairwise_table(fragments(), CFG, engine=eng)
        assert len(eng.gather_cache) == 4
        assert table_digest(t1) == table_digest(t2) == table_digest(t)
        q.put((rank, table_digest(t)))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def single_table():
    return mosaic.build_pairwise_table(fragments(), CFG, engine=OracleEngine(CFG))


def sequential_table(imgs):
    eng = OracleEngine(CFG)
    prep = [eng.prepare([im]) for im in imgs]
    want = mosaic.PairwiseTransformTable(n=len(imgs))
    for a in range(len(imgs)):
        for b in range(a + 1, len(imgs)):
            pa, pb = prep[a], prep[b]
            ok, th, tx, ty, ni = eng.register(pa[0][0], pa[1][0], pa[2][0], int(pa[3][0]), pb[0][0], pb[1][0],
                                              pb[2][0], int(pb[3][0]), pair_seed(CFG.seed, a, b))
            if ok:
                from paper_2405_08578_b200.records import RigidTransform
                want.set_pair(a, b, RigidTransform(th, tx, ty).inverse(), ni)
    return want


def test_single_rank_table_matches_sequential_reference_semantics(single_table):
    want = sequential_table(fragments())
    assert table_digest(single_table) == table_digest(want)
    assert len(single_table.entries) >= 8  # the overlapping neighbours register


def test_mixed_size_images_one_and_two_ranks():
    want = table_digest(sequential_table(mixed_fragments()))
    assert want, "some mixed-size pairs register"
    assert table_digest(mosaic.build_pairwise_table(mixed_fragments(), CFG, engine=OracleEngine(CFG))) == want
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, True)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for rank, dig in (q.get(timeout=10) for _ in procs):
        assert dig == want, f"rank {rank} table differs"


def test_two_ranks_gloo_equal_one_rank(single_table):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    got = [q.get(timeout=10) for _ in procs]
    want = table_digest(single_table)
    for rank, dig in got:
        assert dig == want, f"rank {rank} table differs"


def test_plan_mosaic_places_all_fragments(single_table):
    ids = [f"f{k}" for k in range(single_table.n)]
    plan, placed = mosaic.plan_mosaic(single_table, ids)
    assert plan.final_unmatched == [] and len(placed) == single_table.n
    assert len(plan.rounds) == 1
