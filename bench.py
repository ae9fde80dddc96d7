#!/usr/bin/env python
"""Benchmark of the B200 LP-SIFT hot path -- BASELINE.json configs[1] (C2).

Workload (BASELINE.json configs[1]): 64 seeded 2688x1600
uint8 noise+shapes scenes, LP-SIFT scales L in {8,16,32,64,128}, multiscale
extremum detection + float32 128-d descriptors (no matching).  One step =
detect + describe of the whole 64-image batch; metric Mpixel/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

* ``value``: device-resident inputs, CUDA events around exactly K steps,
  barrier + synchronize on both sides, max over ranks.  Weak scaling: every
  rank describes its own seeded 64-image batch (no collective on the data
  path).  The 275 MB input batch is larger than the 126 MB L2, so no flush.
* ``e2e``: the same metric through the public host API
  (``pipeline.BatchPreparer``): pinned host images in, host keypoints and
  float32 descriptors out, H2D/D2H inside the timed region.
* ``roofline``: the dominant kernel (describe) against measured HBM
  bandwidth (the contract's bound) and against instruction issue (what
  bounds it: warp instructions per launch from the committed ncu capture over
  the live time), plus the detect kernel, from CUDA events inside the timed
  run; ``kernels.describe_precise_f64`` times the float64 kernels.
* ``cpu_baseline``: the oracle port (oracle/lpsift_oracle.py, numpy, the
  reference's algorithm) on this host's cores, bounded sample, rank 0, N=1.
* ``--impl reference``: times that CPU port as the reference arm.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

N_IMAGES, NR, NC = 64, 1600, 2688
SCALES = (8, 16, 32, 64, 128)
WORKLOAD = ("C2: 64 seeded 2688x1600 uint8 noise+shapes scenes; LP-SIFT L in {8..128}; "
            "detect + float32 128-d describe")
CPU_SAMPLE_KP = 6000  # keypoints described per CPU-baseline worker per step


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--images", type=int, default=N_IMAGES)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-match", action="store_true", help="skip the C4 matching measurement")
    ap.add_argument("--no-stitch", action="store_true", help="skip the C3 nine-image stitch measurement")
    ap.add_argument("--no-pairs", action="store_true", help="skip the C5 pairs/s measurement")
    ap.add_argument("--no-composite", action="store_true", help="skip the C3 composite measurement")
    ap.add_argument("--profile-steps", type=int, default=0, help="(ncu) run N steps untimed and exit")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def tensor_peak():
    pj = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(pj):
        with open(pj) as f:
            return float(json.load(f)["bf16_tflops"]), "measured"
    return 1641.9, "fallback"


def pair_phase_evidence(geng, pair_rows, count_launches, reps=10):
    """Device time of a GraphEngine's pair-phase graph (every pair's match ->
    point gather -> RANSAC; CUDA events over back-to-back replays), the
    library kernels one such phase launches (counted on an eager run:
    ``count_launches()``), and the phase's tensor roofline: algorithmic
    2 * 128 * n_a * n_b FLOPs of the pairs' distance matrices (what the
    reference's _distance_matrix computes per pair) over the phase time.  The
    tensor-core kernel b_topk (two passes) is 60-65 % of the serialised phase
    (profiles/r02c_launches_c5_pairs.txt); the rest is certification,
    grouping / tiling and RANSAC."""
    import torch

    g = next(iter(geng._pair_graphs.values()))[0]
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = 2.0 * 128 * sum(float(a) * float(b) for a, b in pair_rows)
    peak, src = tensor_peak()
    ach = flops / (ms / 1e3) / 1e12
    return {"pair_phase_ms": round(ms, 4), "pair_phase_launches": int(count_launches()),
            "roofline": {"bound": "tensor", "kernel": "pair phase (b_topk tcgen05 passes + certification + RANSAC)",
                         "achieved": round(ach, 2), "peak": peak, "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                         "peak_source": src, "algorithmic_flops": flops,
                         "note": "algorithmic 2*128*n_a*n_b per pair over the pair-phase graph replay (CUDA events)"}}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port, bounded sample
# ---------------------------------------------------------------------------

def _cpu_job(args):
    seed, n_kp = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import lpsift_oracle as O
    from paper_2405_08578_b200 import scenes

    img = scenes.scene(NR, NC, seed)
    t0 = time.perf_counter()
    P = O.ramp(img.astype(np.float64), O.default_alpha(NR, NC))
    kp = O.detect(P, SCALES)
    t1 = time.perf_counter()
    O.describe(P, kp[:n_kp], 0.0625, 4, 128, True)
    t2 = time.perf_counter()
    # extrapolated seconds for the whole image: detect + describe of all keypoints
    return (t1 - t0) + (t2 - t1) * len(kp) / n_kp


def cpu_baseline(steps=1, warmup=0, n_kp=CPU_SAMPLE_KP):
    """Mpx/s of the oracle port with one process per host core."""
    import multiprocessing as mp

    P = os.cpu_count() or 1
    vals = []
    with mp.get_context("fork").Pool(P) as pool:
        for s in range(warmup + steps):
            t0 = time.perf_counter()
            secs = pool.map(_cpu_job, [(k, n_kp) for k in range(P)])
            wall = time.perf_counter() - t0
            if s >= warmup:
                # P images processed concurrently; per-image time extrapolated
                vals.append(P * NR * NC / 1e6 / max(secs))
            _ = wall
    return dict(value=float(statistics.median(vals)), unit="Mpixel/s", cores=P, kind="port",
                sample=(f"{P} processes x 1 image each: full detect + describe of the first {n_kp} of "
                        f"134400 keypoints, describe time extrapolated x{134400 / n_kp:.1f}; oracle port "
                        f"(numpy) of the reference algorithm"))


# ---------------------------------------------------------------------------
# C4 matching (BASELINE.json configs[3]): pair-matches/s on tensor cores
# ---------------------------------------------------------------------------

def _cpu_match_job(args):
    """Oracle port: exact float64 MNN matching of an m x m sub-block."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    a, b = args
    from oracle import lpsift_oracle as O

    t0 = time.perf_counter()
    O.match(a, b)
    return a.shape[0] * b.shape[0] / (time.perf_counter() - t0)


def bench_c4_matching(args, world=1, rank=0, dev=None, with_cpu=True, steps=5):
    import torch
    import torch.distributed as dist

    from paper_2405_08578_b200 import device, scenes
    from paper_2405_08578_b200.records import DescriptorConfig
    from paper_2405_08578_b200.rowshard import match_rows_sharded

    a, b = scenes.config4_pair(0)
    cfg = DescriptorConfig(0.0625, 4, 36, True)  # L = 36 (literal {4,8,16} is rejected)
    ds = []
    for im in (a, b):
        t = torch.from_numpy(im).cuda()
        kp = device.detect(t, (36,), meta=False)
        ds.append(device.describe(t, kp, cfg, scale_set=(36,))[0])
        del t
    n1, n2 = ds[0].shape[0], ds[1].shape[0]
    lo, hi = (rank * n1) // world, ((rank + 1) * n1) // world  # my row block of A

    def once():
        if world == 1:
            return device.match(ds[0], ds[1])
        return match_rows_sharded(ds[0][lo:hi], lo, ds[1], 0.35)

    for _ in range(2):
        r = once()
    torch.cuda.synchronize()
    times = []
    for _ in range(steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = once()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = t.item()
        times.append(dt)
    ms = statistics.median(times)
    flops = 2.0 * n1 * n2 * 128
    stats = device.match_stats() if world == 1 else {}
    peak = 1641.9
    pj = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(pj):
        with open(pj) as f:
            peak = float(json.load(f)["bf16_tflops"])
    out = {"metric": "pair-matches/s (C4, 2x 8192x8192 crops, L=36, 128-d MNN, delta_s 0.35)",
           "value": n1 * n2 / (ms / 1e3), "unit": "pair-matches/s", "ms_per_pair": round(ms, 3),
           "n1": n1, "n2": n2, "matches": int(r[0].shape[0]),
           "roofline": {"bound": "tensor",
                        "achieved": round(stats.get("mma_flops", 0) / (ms / 1e3) / 1e12, 2), "peak": peak,
                        "unit": "TFLOP/s", "frac": round(stats.get("mma_flops", 0) / (ms / 1e3) / 1e12 / peak, 4),
                        "note": ("executed fp16 tcgen05 FLOPs (issued MMA tiles) over the whole match call; the "
                                 "duplicate-row grouping removes most of the nominal 2*n1*n2*128")},
           "algorithmic_tflops_equivalent": round(flops / (ms / 1e3) / 1e12, 2),
           "tmem_roofline": tmem_roofline(stats.get("mma_flops", 0), ms, dev),
           "tc_stats": stats,
           "exactness": "bit-exact vs float64 reference arithmetic (tests/test_gpu_parity.py P3)",
           "n_gpus": world, "parallelism": ("single GPU" if world == 1 else
                                            f"rows of A sharded over {world} ranks; NCCL all-reduce of candidate "
                                            "columns and of packed column minima (rowshard.py)"),
           "timing": "host wall clock around the match call, CUDA-synchronized, max over ranks"}
    if with_cpu:
        import multiprocessing as mp

        m = 2000
        A = ds[0][:m].double().cpu().numpy()
        B = ds[1][:m].double().cpu().numpy()
        P = os.cpu_count() or 1
        with mp.get_context("fork").Pool(P) as pool:
            rates = pool.map(_cpu_match_job, [(A, B)] * P)
        out["cpu_baseline"] = {"value": float(sum(rates)), "unit": "pair-matches/s", "cores": P, "kind": "port",
                               "sample": f"{P} processes x exact MNN of a {m}x{m} sub-block (oracle port)"}
    return out


# ---------------------------------------------------------------------------
# C3 nine-image stitch (BASELINE.json configs[2]): seconds at N GPUs
# ---------------------------------------------------------------------------

def bench_c3_stitch(args, world, rank, dev, steps=3, with_cpu=False):
    import torch
    import torch.distributed as dist

    from paper_2405_08578_b200 import mosaic, scenes
    from paper_2405_08578_b200.pipeline import PipelineConfig

    images, truth = scenes.config3_images(0)
    images = [torch.from_numpy(np.ascontiguousarray(im)).pin_memory() for im in images]  # host inputs, pinned
    ids = [f"img{k}" for k in range(9)]
    cfg = PipelineConfig(window_min=32, window_max=128, ransac_iters=2000, ransac_tol=3.0)
    def timed(engine):
        mosaic.build_pairwise_table(images, cfg, engine=engine)  # warm-up (all ranks)
        times = []
        for _ in range(steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            table = mosaic.build_pairwise_table(images, cfg, engine=engine)
            plan, placed = mosaic.plan_mosaic(table, ids)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([dt], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = t.item()
            times.append(dt)
        return statistics.median(times), table, plan, placed

    t_pp, table1, _, _ = timed(mosaic.GpuEngine(cfg, batched=False))
    t_b, table2, _, _ = timed(mosaic.GpuEngine(cfg))
    geng = mosaic.GraphEngine(cfg)
    t_g, table, plan, placed = timed(geng)
    # a rig streaming new frames: a different image set every step through the same engine:
    # the graphs are keyed on shapes, slot addresses and per-image counts -- with the count law of nested
    # scale sets the counts are fixed, so new frames replay the captured graphs (no re-capture)
    alt = [torch.from_numpy(np.ascontiguousarray(im)).pin_memory() for im in scenes.config3_images(1)[0]]
    n_graphs = (len(geng._prep_graphs), len(geng._pair_graphs))
    t_alt = []
    for k in range(4):
        ims = alt if k % 2 else images
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mosaic.plan_mosaic(mosaic.build_pairwise_table(ims, cfg, engine=geng), ids)
        torch.cuda.synchronize()
        t_alt.append(time.perf_counter() - t0)
    recaptured = (len(geng._prep_graphs), len(geng._pair_graphs)) != n_graphs
    from paper_2405_08578_b200 import _lib

    def c3_launches():  # library kernels of one eager pair phase (the graph replays the same sequence)
        eng = mosaic.GpuEngine(cfg)
        rows, cols, desc, cnt = eng.prepare(images[:9])
        h = cnt.cpu().tolist()
        items = [(rows[a], cols[a], desc[a], h[a], rows[b], cols[b], desc[b], h[b], 0)
                 for a in range(9) for b in range(a + 1, 9)]
        torch.cuda.synchronize()
        l0 = _lib.kernel_launches()
        eng._pairs_dev(items)
        torch.cuda.synchronize()
        return _lib.kernel_launches() - l0

    cnt9 = geng.prepare(images)[3].cpu().tolist()
    phase = pair_phase_evidence(geng, [(cnt9[a], cnt9[b]) for a in range(9) for b in range(a + 1, 9)], c3_launches)
    assert table.entries.keys() == table1.entries.keys() == table2.entries.keys()
    n_pairs = len(table.entries) // 2
    # control (untimed): the same generator with the perturbations off registers the overlapping pairs --
    # the timed set registers none because LP-SIFT's window peaks do not survive its rotation / noise
    # (the live reference agrees pair by pair: tests/test_gpu_pairs.py, goldens from tests/golden/make_golden.py)
    ctl_images, _ = scenes.config3_images(0, rot_deg=0.0, scale_range=(1.0, 1.0), noise=0.0)
    ctl = mosaic.build_pairwise_table(ctl_images, cfg)
    _, ctl_placed = mosaic.plan_mosaic(ctl, ids)
    cpu = None
    if with_cpu and rank == 0:
        import multiprocessing as mp

        P = os.cpu_count() or 1
        host = [im.numpy() for im in images]
        with mp.get_context("fork").Pool(P) as pool:
            ch = oracle_pair_chain(pool, P, host[0], host[1], (32, 64, 128), 128, 2000, 0)
        core_s = 9 * float(np.mean(ch["prepare_core_s"])) + 36 * (ch["match_core_s"] + ch["ransac_s"])
        cpu = {"value": round(core_s / P, 3), "unit": "s", "cores": P, "kind": "port",
               "sample": (f"oracle port chain of pair (0, 1) (2 images prepared, exact float64 MNN of "
                          f"{ch['n_kp'][0]}x{ch['n_kp'][1]} split over {P} processes, RANSAC 2000 it.); the table "
                          f"= 9 prepares + 36 pairs extrapolated from its core-seconds ({core_s:.1f}) / {P} cores, "
                          f"perfect parallel scaling assumed"),
               "pair_matches": ch["matches"], "pair_registered": ch["registered"]}
    return {"metric": "9-image stitch seconds (C3: detect/describe 9 x 2688x1600, 36 pairs match + RANSAC, plan)",
            "value": round(t_g, 4), "unit": "s", "higher_is_better": False,
            "batched_eager_value": round(t_b, 4), "per_pair_calls_value": round(t_pp, 4),
            "alternating_frames_value": round(statistics.median(t_alt[1:]), 4), "alternating_frames_recaptured": recaptured,
            "batching": "value: mosaic.GraphEngine -- the 9 images (pinned host memory) uploaded every step, "
                        "detect+describe replayed as CUDA graphs (3-image chunks, uploads overlapped), the whole "
                        "pair phase (36 pairs: ps_match_batch_async -- every image's descriptor set grouped and "
                        "tiled once, one launch per stage for all pairs -- then ps_register_batch_async, the match "
                        "counts feeding RANSAC on the device) replayed as one graph, one result read; "
                        "batched_eager_value: the same chain launched eagerly; per_pair_calls_value: one "
                        "synchronous pair at a time",
            **phase,
            "n_gpus": world, "registered_pairs": n_pairs, "placed": len(placed),
            "rounds": len(plan.rounds), "unmatched": plan.final_unmatched,
            "control_translation_only_noise0": {"registered_pairs": len(ctl.entries) // 2, "placed": len(ctl_placed)},
            "timing": "host wall clock around the whole call, CUDA-synchronized, max over ranks",
            "e2e": {"value": round(t_g, 4), "unit": "s", "h2d_bytes_per_step": int(sum(im.numel() for im in images)),
                    "d2h_bytes_per_step": 36 * 8 * 8,
                    "api": "mosaic.build_pairwise_table + plan_mosaic from pinned host images"},
            "cpu_baseline": cpu,
            "parallelism": f"images then pairs sharded over {world} rank(s); NCCL all-gather of keypoint/descriptor "
                           "slots and of the pair results"}


# ---------------------------------------------------------------------------
# C3 composite: the nine crops warped into one canvas
# ---------------------------------------------------------------------------

def c3_placements():
    """The nine C3 crops placed rigidly by their generator truth (rotation
    about the crop centre onto the source frame; the +-5 % scale is ignored)."""
    from paper_2405_08578_b200 import compositor as K, scenes
    from paper_2405_08578_b200.records import RigidTransform

    images, truth = scenes.config3_images(0)
    ids, pl = [], []
    for k, (img, (r0, c0, th, _)) in enumerate(zip(images, truth)):
        h, w = img.shape
        hx, hy = (w - 1) / 2.0, (h - 1) / 2.0
        c, s = math.cos(th), math.sin(th)
        tx = c0 + hx - (c * hx - s * hy)
        ty = r0 + hy - (s * hx + c * hy)
        ids.append(f"img{k}")
        pl.append(K.Placement(f"img{k}", RigidTransform(th, tx, ty)))
    return dict(zip(ids, images)), pl


def bench_c3_composite(args, rank, dev, with_cpu, steps=5):
    """Feather + bilinear composite of the nine C3 crops on one GPU (rank 0;
    the canvas is one output, no data-path collective)."""
    import torch

    from paper_2405_08578_b200 import compositor as K

    if rank != 0:
        return None
    images, pl = c3_placements()
    canvas = K.compute_canvas(pl, {k: v.shape for k, v in images.items()})
    dimg = {k: torch.from_numpy(v).to(dev) for k, v in images.items()}
    for _ in range(2):
        K.warp_and_blend_device(dimg, pl, canvas)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        K.warp_and_blend_device(dimg, pl, canvas)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    npx = canvas.width * canvas.height
    nbytes = 16 * npx + sum(v.size for v in images.values())  # pixels + weightmap out, every source read once
    peak, _ = measured_peaks()
    out = {"metric": "canvas Mpixel/s (C3 composite: 9 x 2688x1600 u8 crops, feather, bilinear, float64 canvas)",
           "value": round(npx / 1e6 / (ms / 1e3), 1), "unit": "Mpixel/s", "ms": round(ms, 4),
           "canvas_hw": [canvas.height, canvas.width], "placements": len(pl),
           "roofline": {"bound": "hbm", "achieved": round(nbytes / (ms / 1e3) / 1e9, 1), "peak": peak,
                        "unit": "GB/s", "frac": round(nbytes / (ms / 1e3) / 1e9 / peak, 4),
                        "algorithmic_bytes": nbytes},
           "exactness": "bit-identical to the reference warp_and_blend (tests/test_gpu_parity.py)",
           "timing": "CUDA events, inputs resident"}
    if with_cpu:
        from oracle import lpsift_oracle as O

        row = [k for k in images][:3]  # one grid row of crops: bounded CPU sample
        tr = [(p.transform.theta, p.transform.t_x, p.transform.t_y) for p in pl if p.image_id in row]
        imgs = [images[k] for k in row]
        bounds = O.canvas_bounds(tr, [a.shape for a in imgs])
        t0 = time.perf_counter()
        O.composite(imgs, tr, bounds)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": round(bounds[0] * bounds[1] / 1e6 / dt, 2), "unit": "Mpixel/s", "cores": 1,
                               "kind": "port", "sample": f"oracle composite of 3 of the 9 crops "
                               f"({bounds[1]}x{bounds[0]} canvas), numpy, one process"}
    return out


# ---------------------------------------------------------------------------
# K4 RANSAC: hypothesis-pair evaluations per second
# ---------------------------------------------------------------------------

def bench_ransac(args, rank, dev, with_cpu, n=1000, iters=2000, steps=5):
    """Seeded correspondences (60 % inliers of a rigid motion + 1 px noise,
    40 % uniform outliers): iterations x n transfer errors per call."""
    import torch

    from paper_2405_08578_b200 import device

    if rank != 0:
        return None
    rng = np.random.default_rng(7)
    src = rng.uniform(0, 1000, size=(n, 2))
    th, t = 0.2, np.array([35.0, -12.0])
    R = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
    dst = src @ R.T + t + rng.normal(0, 1.0, size=(n, 2))
    out = rng.random(n) < 0.4
    dst[out] = rng.uniform(0, 1000, size=(int(out.sum()), 2))
    s_d, d_d = torch.from_numpy(src).to(dev), torch.from_numpy(dst).to(dev)
    for _ in range(2):
        device.ransac(s_d, d_d, iters, 3.0, 8, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        r = device.ransac(s_d, d_d, iters, 3.0, 8, 0)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    res = {"metric": "RANSAC hypothesis-pair evaluations/s (2-point rigid, n=1000, 2000 iterations)",
           "value": round(iters * n / dt, 1), "unit": "evaluations/s", "ms_per_call": round(dt * 1e3, 4),
           "consensus": int(r.consensus), "inliers": int(len(r.inliers)),
           "timing": "host wall clock per device.ransac call (includes the host PCG64 sample stream and the "
                     "result read-back), CUDA-synchronized"}
    if with_cpu:
        from oracle import lpsift_oracle as O

        t0 = time.perf_counter()
        O.ransac(src, dst, iters, 3.0, 8, 0)
        c = time.perf_counter() - t0
        res["cpu_baseline"] = {"value": round(iters * n / c, 1), "unit": "evaluations/s", "cores": 1,
                               "kind": "port", "sample": "the same call, numpy oracle port, one process"}
    return res


# ---------------------------------------------------------------------------
# C5 illumination pairs (BASELINE.json configs[4]): pairs/s
# ---------------------------------------------------------------------------

def bench_c5_pairs(args, world, rank, dev, n_pairs=256, steps=2, with_cpu=False):
    """Full path per pair (detect, describe both images; match; RANSAC) on
    the RGB pixels: BT.601 grey through the device ingest path (integer luma
    key for detection, the run host's grey table for values and the
    descriptor raster -- bit-identical to load_image's to_grayscale);
    pairs sharded over ranks, no collective on the data path."""
    import torch
    import torch.distributed as dist

    from paper_2405_08578_b200 import device, scenes
    from paper_2405_08578_b200.pipeline import PipelineConfig

    cfg = PipelineConfig(window_min=16, window_max=64)
    from paper_2405_08578_b200 import shard

    mine = shard.round_robin(n_pairs, rank, world)  # pairs sharded, no data-path collective
    grey = []
    import multiprocessing as mp

    with mp.get_context("fork").Pool(max(1, min(16, (os.cpu_count() or 1) // max(world, 1)))) as pool:
        for a, b in pool.imap(scenes._c5_job, mine):
            grey.append(device.as_device_images(torch.from_numpy(np.stack([a, b])).to(dev), rgb=True))
    sizes, dcfg = cfg.scale_set().sizes, cfg.descriptor_config()

    def run_pair(g):
        kp = device.detect(g, sizes, meta=False)
        d = device.describe(g, kp, dcfg, scale_set=kp.scale_set)
        r1, r2, _ = device.match(d[0][: kp.cap], d[1][: kp.cap])
        n = int(r1.shape[0])
        ok = False
        if n >= cfg.min_inliers:
            src, dst = device.pair_points(r1, r2, kp.row[0], kp.col[0], kp.row[1], kp.col[1])
            ok = device.ransac(src, dst, cfg.ransac_iters, cfg.ransac_tol, cfg.min_inliers, cfg.seed).ok
        return n, ok

    # batched: every local image detected + described in one call, all pairs
    # matched with one count read-back, all RANSAC runs with one result read
    allimg = device.as_device_images(torch.cat([g.data for g in grey]), rgb=True) if grey else None
    streams = [torch.cuda.Stream(dev) for _ in range(4)]

    def run_batched():
        if allimg is None:
            return []
        kp = device.detect(allimg, sizes, meta=False)
        d = device.describe(allimg, kp, dcfg, scale_set=kp.scale_set)
        ms = device.match_many([(d[2 * q], d[2 * q + 1]) for q in range(len(grey))], cfg.delta_s, streams=streams)
        jobs, where = [], []
        for q, (r1, r2, _) in enumerate(ms):
            if int(r1.shape[0]) >= cfg.min_inliers:
                src, dst = device.pair_points(r1, r2, kp.row[2 * q], kp.col[2 * q], kp.row[2 * q + 1],
                                              kp.col[2 * q + 1])
                jobs.append((src, dst, cfg.ransac_iters, cfg.ransac_tol, cfg.min_inliers, cfg.seed))
                where.append(q)
        ok = [False] * len(ms)
        for q, o in zip(where, device.ransac_many(jobs, streams=streams)):
            ok[q] = o.ok
        return [(int(m[0].shape[0]), k) for m, k in zip(ms, ok)]

    def timed(fn):
        out = fn()  # warm-up
        times = []
        for _ in range(steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = fn()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([dt], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = t.item()
            times.append(dt)
        return statistics.median(times), out

    from paper_2405_08578_b200 import mosaic
    from paper_2405_08578_b200.pipeline import pair_seed  # noqa: F401

    geng = mosaic.GraphEngine(cfg, n_streams=8)

    def run_graph():
        if allimg is None:
            return []
        rows, cols, desc, cnt = geng.prepare_device(allimg)
        h = cnt.cpu().tolist()
        R, Cc, Dd = rows.unbind(0), cols.unbind(0), desc.unbind(0)  # per-image views in one call each
        items = [(R[2 * q], Cc[2 * q], Dd[2 * q], h[2 * q], R[2 * q + 1], Cc[2 * q + 1], Dd[2 * q + 1],
                  h[2 * q + 1], cfg.seed) for q in range(len(grey))]
        return [(None, o[0]) for o in geng.register_many(items)]

    # e2e: the RGB pairs from pinned host memory, uploaded inside the timed region
    host_rgb = torch.cat([g.data for g in grey]).cpu().pin_memory() if grey else None
    dev_rgb = torch.empty_like(host_rgb, device=dev) if grey else None
    e2e_img = device.as_device_images(dev_rgb, rgb=True) if grey else None

    def run_graph_e2e():
        if e2e_img is None:
            return []
        dev_rgb.copy_(host_rgb, non_blocking=True)
        rows, cols, desc, cnt = geng.prepare_device(e2e_img)
        h = cnt.cpu().tolist()
        R, Cc, Dd = rows.unbind(0), cols.unbind(0), desc.unbind(0)
        items = [(R[2 * q], Cc[2 * q], Dd[2 * q], h[2 * q], R[2 * q + 1], Cc[2 * q + 1], Dd[2 * q + 1],
                  h[2 * q + 1], cfg.seed) for q in range(len(grey))]
        return [(None, o[0]) for o in geng.register_many(items)]

    n_sub = min(len(grey), 16)  # the one-pair-at-a-time variant on a bounded subset
    dt1, stats1 = timed(lambda: [run_pair(g) for g in grey[:n_sub]])
    dtb, stats = timed(run_batched)
    dt, statsg = timed(run_graph)
    dte, statse = timed(run_graph_e2e)
    from paper_2405_08578_b200 import _lib

    def c5_launches():  # library kernels of one eager pair phase (the graph replays the same sequence)
        eng = mosaic.GpuEngine(cfg)
        rows, cols, desc, cnt = eng._prepare_dev(allimg)
        h = cnt.cpu().tolist()
        items = [(rows[2 * q], cols[2 * q], desc[2 * q], h[2 * q], rows[2 * q + 1], cols[2 * q + 1],
                  desc[2 * q + 1], h[2 * q + 1], cfg.seed) for q in range(len(grey))]
        torch.cuda.synchronize()
        l0 = _lib.kernel_launches()
        eng._pairs_dev(items)
        torch.cuda.synchronize()
        return _lib.kernel_launches() - l0

    phase = {}
    if grey:
        cn = geng.prepare_device(allimg)[3].cpu().tolist()
        phase = pair_phase_evidence(geng, [(cn[2 * q], cn[2 * q + 1]) for q in range(len(grey))], c5_launches)
    assert [s[1] for s in statse] == [s[1] for s in statsg]
    assert [s[0] for s in stats[:n_sub]] == [s[0] for s in stats1]
    assert [s[1] for s in stats[:n_sub]] == [s[1] for s in stats1] and [s[1] for s in statsg] == [s[1] for s in stats]
    return {"metric": "pairs/s (C5: 1920x1080 RGB pairs, BT.601 grey, homography warp + gain/offset/noise, "
                      "L 16..64, full detect/describe/match/RANSAC)",
            "value": round(n_pairs / dt, 3), "unit": "pairs/s", "pairs": n_pairs, "n_gpus": world,
            "per_pair_calls_value": round(n_sub * world / dt1, 3), "batched_eager_value": round(n_pairs / dtb, 3),
            "mean_matches": float(np.mean([s[0] for s in stats])) if stats else 0.0,
            "registered": int(sum(s[1] for s in stats)),
            "timing": "host wall clock, CUDA-synchronized, max over ranks; RGB inputs resident on the GPU",
            "batching": "value: mosaic.GraphEngine -- all local images detected + described in one replayed "
                        "CUDA graph, one count read, then the pair phase replayed as one graph: "
                        "ps_match_batch_async (every pair's match, one launch per stage) and "
                        "ps_register_batch_async (every pair's point gather + RANSAC on the device-side counts), "
                        "one result read; batched_eager_value: detect/describe in one call, per-pair matcher and "
                        "RANSAC launches over 4 streams with one count and one result read-back; "
                        "per_pair_calls_value: one synchronous pair at a time (first 16 pairs of each rank)",
            **phase,
            "ingest": "RGB8 pixel type: luma-key detection, host-built 2^24 grey table (ingest.py)",
            "e2e": {"value": round(n_pairs / dte, 3), "unit": "pairs/s",
                    "h2d_bytes_per_step": int(host_rgb.numel()) * world if grey else 0,
                    "d2h_bytes_per_step": n_pairs * 8 * 8,
                    "api": "pinned host RGB pairs uploaded each step, then the GraphEngine chain (prepare_device "
                           "+ register_many), success flags read back"},
            "cpu_baseline": _c5_cpu(world, rank) if with_cpu else None}


def _c5_cpu(world, rank):
    """Oracle-port chain of C5 pair 0 on this host's cores, extrapolated to pairs/s."""
    if rank != 0 or world != 1:
        return None
    import multiprocessing as mp

    from paper_2405_08578_b200 import scenes

    a, b, _ = scenes.config5_pair(0)
    P = os.cpu_count() or 1
    with mp.get_context("fork").Pool(P) as pool:
        ch = oracle_pair_chain(pool, P, a, b, (16, 32, 64), 64, 2000, 0)
    core_s = sum(ch["prepare_core_s"]) + ch["match_core_s"] + ch["ransac_s"]
    return {"value": round(P / core_s, 4), "unit": "pairs/s", "cores": P, "kind": "port",
            "sample": (f"oracle port chain of C5 pair 0 (BT.601 grey, 2 images prepared, exact float64 MNN of "
                       f"{ch['n_kp'][0]}x{ch['n_kp'][1]} split over {P} processes, RANSAC 2000 it.): "
                       f"{core_s:.1f} core-seconds per pair -> pairs/s = {P} cores / that, perfect scaling assumed"),
            "pair_matches": ch["matches"], "pair_registered": ch["registered"]}


# ---------------------------------------------------------------------------
# CPU oracle chain for one pair (C1 latency, C3 / C5 baselines): prepare each
# image on one core, the exact float64 MNN match split by row blocks over P
# processes (column minima merged with the first-occurrence rule), RANSAC
# on one core.  Timed per part so per-config totals can be stated.
# ---------------------------------------------------------------------------

def _oracle_prepare_job(args):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import lpsift_oracle as O

    img, scales, l_max = args
    t0 = time.perf_counter()
    grey = img.astype(np.float64) if img.ndim == 2 else img.astype(np.float64) @ np.array([0.299, 0.587, 0.114])
    P = O.ramp(grey, O.default_alpha(*grey.shape))
    kp = O.detect(P, scales)
    desc = O.describe(P, kp, 0.0625, 4, l_max, True)
    return kp, desc, time.perf_counter() - t0


def _oracle_rows_job(args):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import lpsift_oracle as O

    A, B, i0 = args
    t0 = time.perf_counter()
    n2 = B.shape[0]
    nn = np.empty(A.shape[0], np.int64)
    best = np.empty(A.shape[0])
    cbest, carg = np.full(n2, np.inf), np.zeros(n2, np.int64)
    for j0, D in O.distances(A, B):
        j = np.argmin(D, axis=1)
        nn[j0:j0 + len(j)] = j
        best[j0:j0 + len(j)] = D[np.arange(len(j)), j]
        ci = np.argmin(D, axis=0)
        cv = D[ci, np.arange(n2)]
        upd = cv < cbest
        cbest[upd], carg[upd] = cv[upd], ci[upd] + j0 + i0
    return i0, nn, best, cbest, carg, time.perf_counter() - t0


def oracle_pair_chain(pool, P, img_a, img_b, scales, l_max, iters, seed):
    """The oracle port's chain for one pair -> timings and outcome."""
    from oracle import lpsift_oracle as O

    t0 = time.perf_counter()
    (ka, da, ta), (kb, db, tb) = pool.map(_oracle_prepare_job, [(img_a, scales, l_max), (img_b, scales, l_max)])
    t1 = time.perf_counter()
    da32, db32 = da.astype(np.float32).astype(np.float64), db.astype(np.float32).astype(np.float64)
    n1 = len(da32)
    cuts = [(n1 * k) // P for k in range(P + 1)]
    parts = pool.map(_oracle_rows_job, [(da32[cuts[k]:cuts[k + 1]], db32, cuts[k]) for k in range(P)
                                        if cuts[k + 1] > cuts[k]])
    nn12, best12 = np.concatenate([p[1] for p in parts]), np.concatenate([p[2] for p in parts])
    cbest, carg = parts[0][3].copy(), parts[0][4].copy()
    for p in parts[1:]:  # blocks in row order: strict < keeps the earliest row on ties
        upd = p[3] < cbest
        cbest[upd], carg[upd] = p[3][upd], p[4][upd]
    rows = np.arange(n1)
    ok = (carg[nn12] == rows) & (best12 < 0.35)
    r1, r2, dl = rows[ok], nn12[ok], best12[ok]
    order = np.lexsort((r2, r1, dl))
    r1, r2 = r1[order], r2[order]
    t2 = time.perf_counter()
    registered = False
    if len(r1) >= 8:
        try:
            O.ransac(*O.pair_points(r1, r2, ka, kb), iters, 3.0, 8, seed)
            registered = True
        except O.NoConsensus:
            pass
    t3 = time.perf_counter()
    return {"prepare_core_s": [ta, tb], "match_core_s": float(sum(p[5] for p in parts)), "ransac_s": t3 - t2,
            "wall_s": t3 - t0, "prepare_wall_s": t1 - t0, "match_wall_s": t2 - t1, "matches": int(len(r1)),
            "registered": registered, "n_kp": [len(ka), len(kb)]}


# ---------------------------------------------------------------------------
# C1 latency (BASELINE.json configs[0]): one pair through the whole chain
# ---------------------------------------------------------------------------

def bench_c1_latency(args, rank, dev, with_cpu, steps=10):
    """Device latency (crops resident, detect+describe both, MNN match,
    RANSAC 1000 it., result read) and e2e latency (host numpy crops in,
    RegistrationResult out, through pipeline.prepare_image /
    register_prepared -- the reference's own call sequence, pipeline.py:171-209);
    the ratio-0.8 strategy (extra) timed on the same descriptors."""
    import torch

    from paper_2405_08578_b200 import device, matcher, pipeline as PL, scenes
    from paper_2405_08578_b200.records import IntensityImage, MatcherConfig

    if rank != 0:
        return None
    a, b = scenes.config1_pair(0)
    cfg = PL.PipelineConfig(window_min=16, window_max=64, ransac_iters=1000, ransac_tol=3.0, seed=0)
    sizes, dcfg = cfg.scale_set().sizes, cfg.descriptor_config()
    ta, tb = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    pair = device.DeviceImages(torch.stack([ta, tb]), "u8", device.default_alpha(*a.shape))

    def dev_once():
        kp = device.detect(pair, sizes, meta=False)
        d = device.describe(pair, kp, dcfg, scale_set=kp.scale_set)
        r1, r2, _ = device.match(d[0], d[1], cfg.delta_s)
        src, dst = device.pair_points(r1, r2, kp.row[0], kp.col[0], kp.row[1], kp.col[1])
        return device.ransac(src, dst, cfg.ransac_iters, cfg.ransac_tol, cfg.min_inliers, cfg.seed), d

    def e2e_once():
        pa = PL.prepare_image(IntensityImage(a, "a"), cfg)
        pb = PL.prepare_image(IntensityImage(b, "b"), cfg)
        return PL.register_prepared(pa, pb, cfg, seed=0)

    def timed(fn):
        for _ in range(3):
            out = fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(ts), out

    ms_dev, (reg, d) = timed(dev_once)
    ms_e2e, (pairs, res, _, _) = timed(e2e_once)
    ms_ratio, rr = timed(lambda: device.match(d[0], d[1], 0.8, "ratio_test"))
    out = {"metric": "C1 pair latency (768x1024 crops, L 16..64, detect+describe both, MNN match, RANSAC 1000)",
           "value": round(ms_dev, 3), "unit": "ms", "higher_is_better": False,
           "matches": int(len(pairs)), "inliers": int(len(reg.inliers)), "registered": bool(reg.ok),
           "t_x": round(float(reg.t_x), 6), "t_y": round(float(reg.t_y), 6),
           "e2e": {"value": round(ms_e2e, 3), "unit": "ms", "api": "pipeline.prepare_image x2 + register_prepared "
                   "(host numpy crops in, host MatchPair list + RegistrationResult out)",
                   "h2d_bytes_per_step": int(a.nbytes + b.nbytes),
                   "d2h_bytes_per_step": int(len(pairs) * (4 * 4 + 8 + 8))},
           "ratio_test_0_8": {"value": round(ms_ratio, 3), "unit": "ms", "matches": int(rr[0].shape[0]),
                              "path": "float64 CUDA-core top-2 (nn_pass<top2> + ratio_select), bit-exact vs its "
                                      "numpy oracle (tests/test_gpu_ratio.py)",
                              "pair_matches_per_s": round(6144 * 6144 / (ms_ratio / 1e3), 1)},
           "timing": "host wall clock per call, CUDA-synchronized, median of %d" % steps}
    if with_cpu:
        import multiprocessing as mp

        P = os.cpu_count() or 1
        with mp.get_context("fork").Pool(P) as pool:
            ch = oracle_pair_chain(pool, P, a, b, (16, 32, 64), 64, 1000, 0)
        out["cpu_baseline"] = {"value": round(ch["wall_s"] * 1e3, 1), "unit": "ms", "cores": P, "kind": "port",
                               "sample": "the whole C1 pair through the oracle port (numpy restatement of the "
                                         "reference): both images prepared in parallel (1 core each), the exact "
                                         f"float64 match split by row blocks over {P} processes, RANSAC on one "
                                         "core; wall clock, not extrapolated",
                               "matches": ch["matches"], "registered": ch["registered"],
                               "parts_s": {"prepare": round(ch["prepare_wall_s"], 3),
                                           "match": round(ch["match_wall_s"], 3), "ransac": round(ch["ransac_s"], 3)}}
    return out


def bench_detect_shapes(dev, peak):
    """K1 on the shapes of C3 (u8, L 32..128), C4 (u8, L = 36) and C5 (RGB8, L 16..64): one
    detect call replayed as a CUDA graph (no host launch gaps), CUDA events over 20 replays."""
    import torch

    from paper_2405_08578_b200 import device

    out = {}
    cases = [("C3 9x1600x2688 u8 L32..128", (9, 1600, 2688), (32, 64, 128), False),
             ("C4 2x8192x8192 u8 L36", (2, 8192, 8192), (36,), False),
             ("C5 64x1080x1920 rgb8 L16..64", (64, 1080, 1920), (16, 32, 64), True)]
    for name, (B, nr, nc), scales, rgb in cases:
        g = torch.Generator(device=dev).manual_seed(1)
        t = torch.randint(0, 256, (B, nr, nc, 3) if rgb else (B, nr, nc), dtype=torch.uint8, device=dev, generator=g)
        im = device.as_device_images(t, rgb=rgb)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                kp = device.detect(im, scales, meta=False, stream=s)
            s.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                kp = device.detect(im, scales, meta=False, stream=s)
            gr.replay()
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(20):
                gr.replay()
            e1.record(s)
            s.synchronize()
        ms = e0.elapsed_time(e1) / 20
        nbytes = t.numel() + int(kp.count.sum()) * 16
        out[name] = {"us": round(ms * 1e3, 1), "GB/s": round(nbytes / ms / 1e6, 1),
                     "frac_hbm": round(nbytes / ms / 1e6 / peak, 4), "bytes_per_launch": nbytes}
        del t, im, kp, gr
    return out


# ---------------------------------------------------------------------------
# Dense tensor-core matching at C4 scale (SURVEY §8(d) K3 >= 50 % of peak)
# ---------------------------------------------------------------------------

def bench_c4_dense(args, rank, dev, steps=5):
    """103,968^2 distinct unit descriptors (half of B near-copies of A rows,
    so half the columns are matchable): the MNN match on the tensor cores,
    algorithmic 2*n1*n2*128 FLOPs / time vs the measured bf16 dense peak.
    ``passes`` reports whether the column pass ran (2) or pass 1's exact
    distances below delta_s decided the columns (1; csrc/match_tc.cu ColCand)."""
    import torch

    from paper_2405_08578_b200 import device

    if rank != 0:
        return None
    n = 103_968
    g = torch.Generator(device=dev).manual_seed(4)
    A = torch.randn((n, 128), generator=g, device=dev)
    A = A / A.norm(dim=1, keepdim=True)
    B = torch.randn((n, 128), generator=g, device=dev)
    B = B / B.norm(dim=1, keepdim=True)
    half = n // 2
    B[:half] = A[torch.randperm(n, generator=g, device=dev)[:half]] + 0.01 * torch.randn((half, 128), generator=g,
                                                                                        device=dev)
    B = B / B.norm(dim=1, keepdim=True)
    A, B = A.float().contiguous(), B.float().contiguous()
    for _ in range(2):
        r = device.match(A, B, 0.35, path="tensor")
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        r = device.match(A, B, 0.35, path="tensor")
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    stats = device.match_stats()
    ex = device.match(A, B, 0.35, path="exact")  # P3 on this data: the exact float64 path, untimed
    same = bool(torch.equal(r[0], ex[0]) and torch.equal(r[1], ex[1]) and torch.equal(r[2], ex[2]))
    flops = 2.0 * n * n * 128
    peak = _bf16_peak()
    return {"metric": "dense MNN pair-matches/s (103,968^2 distinct unit 128-d fp32 descriptors, tcgen05)",
            "value": round(n * n / (ms / 1e3), 1), "unit": "pair-matches/s", "ms_per_pair": round(ms, 3),
            "matches": int(r[0].shape[0]), "exact_equal": same, "passes": stats.get("passes", 0),
            "roofline": {"bound": "tensor", "achieved": round(flops / (ms / 1e3) / 1e12, 1), "peak": peak,
                         "unit": "TFLOP/s", "frac": round(flops / (ms / 1e3) / 1e12 / peak, 4),
                         "algorithmic_flops": flops,
                         "executed_mma_flops": stats.get("mma_flops", 0),
                         "note": "algorithmic 2*n1*n2*128 over the whole call (duplicate grouping, operand "
                                 "tiles, the tensor-core pass(es), the exact float64 certification, the column "
                                 "argmin and the ordering included); executed counts the fp16 MMA tiles "
                                 "issued (K = 144 incl. the |y|^2 augmentation)"},
            "tmem_roofline": tmem_roofline(stats.get("mma_flops", 0), ms, dev),
            "timing": "CUDA events over %d back-to-back calls (each has one host count read)" % steps}


_TMEM_PEAK = {}


def tmem_probe(dev):
    """Tensor-memory read bandwidth of this GPU (ps_probe_tmem_read, CUDA events)."""
    import ctypes as C

    import torch

    from paper_2405_08578_b200 import _lib

    if "gbs" in _TMEM_PEAK:
        return _TMEM_PEAK
    L = _lib.lib()
    sink = torch.zeros(148, dtype=torch.int32, device=dev)
    nb = C.c_double()
    st = torch.cuda.current_stream()
    for _ in range(2):
        _lib.check(L.ps_probe_tmem_read(20000, 148, C.c_void_p(sink.data_ptr()), C.byref(nb),
                                        C.c_void_p(st.cuda_stream)), "probe")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5):
        _lib.check(L.ps_probe_tmem_read(20000, 148, C.c_void_p(sink.data_ptr()), C.byref(nb),
                                        C.c_void_p(st.cuda_stream)), "probe")
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    _TMEM_PEAK.update({"gbs": round(nb.value / (ms / 1e3) / 1e9, 1), "ms": round(ms, 3),
                       "how": "ps_probe_tmem_read: 148 CTAs x 16 warps, two 64-column tcgen05.ld (32x32b.x64) per "
                              "wait x 20000, all 512 TMEM columns allocated per SM, CUDA events"})
    return _TMEM_PEAK


def tmem_roofline(mma_flops, ms, dev):
    """Tensor-memory read traffic of the tensor-core matcher against the
    box's TMEM read bandwidth (ps_probe_tmem_read): the epilogue reads every
    fp32 accumulator once (128 KB per 128 x 256 tile; tiles = executed MMA
    FLOPs / (2 * 128 * 256 * 144)).  The fraction is small: the TMEM read
    is NOT what bounds the kernel (K3 explains what does)."""
    if not mma_flops:
        return None
    pk = tmem_probe(dev)
    tiles = mma_flops / (2.0 * 128 * 256 * 144)
    gbs = tiles * 128 * 256 * 4 / (ms / 1e3) / 1e9
    return {"bound": "tmem-read (not binding)", "achieved": round(gbs, 1), "peak": pk["gbs"], "unit": "GB/s",
            "frac": round(gbs / pk["gbs"], 4), "tiles": int(tiles), "probe": pk}


def _bf16_peak():
    pj = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(pj):
        with open(pj) as f:
            return float(json.load(f)["bf16_tflops"])
    return 2250.0


def fp64_probe(dev):
    """FP64-pipe peak of this GPU (ps_probe_fp64_fma, CUDA events)."""
    import ctypes as C

    import torch

    from paper_2405_08578_b200 import _lib

    L = _lib.lib()
    sink = torch.zeros(148 * 8, dtype=torch.float64, device=dev)
    fl = C.c_double()
    st = torch.cuda.current_stream()
    for _ in range(2):
        _lib.check(L.ps_probe_fp64_fma(20000, 148 * 8, C.c_void_p(sink.data_ptr()), C.byref(fl),
                                       C.c_void_p(st.cuda_stream)), "probe")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5):
        _lib.check(L.ps_probe_fp64_fma(20000, 148 * 8, C.c_void_p(sink.data_ptr()), C.byref(fl),
                                       C.c_void_p(st.cuda_stream)), "probe")
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    return {"tflops": round(fl.value / (ms / 1e3) / 1e12, 2), "ms": round(ms, 3),
            "how": "ps_probe_fp64_fma: 148x8 blocks x 256 threads x 8 independent DFMA chains x 20000 steps, "
                   "CUDA events, 2 FLOPs per DFMA"}



# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, uuid):
        self.uuid, self.proc, self.lines = uuid, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.uuid, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2405_08578_b200 import _lib, device, scenes
    from paper_2405_08578_b200.pipeline import BatchPreparer, PipelineConfig, alloc_host_features
    from paper_2405_08578_b200.records import DescriptorConfig, default_alpha

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    # weak scaling: every rank runs the full C2 batch of its own seeded images
    # (seeds rank*64 .. rank*64+63; rank 0's batch is BASELINE configs[1]'s)
    from paper_2405_08578_b200 import shard

    mine = shard.image_slots(rank, world, args.images)
    n = len(mine)
    host = np.empty((n, NR, NC), dtype=np.uint8)
    import multiprocessing as mp

    with mp.get_context("fork").Pool(min(16, os.cpu_count() or 1)) as pool:
        for i, img in enumerate(pool.imap(scenes._scene_job, [(NR, NC, k) for k in mine])):
            host[i] = img
    alpha = default_alpha(NR, NC)
    cfg = DescriptorConfig(0.0625, 4, 128, True)
    imgs = torch.from_numpy(host).to(dev)
    dimg = device.DeviceImages(imgs, "u8", alpha)
    stream = torch.cuda.current_stream()
    kp = device.detect(dimg, SCALES, meta=False)
    K = kp.cap
    desc = torch.empty((n, K, 128), dtype=torch.float32, device=dev)

    def step(evs=None):
        if evs:
            evs[0].record(stream)
        k = device.detect(dimg, SCALES, meta=False)
        if evs:
            evs[1].record(stream)
        device.describe_into(dimg, k, cfg, desc, scale_set=k.scale_set)
        if evs:
            evs[2].record(stream)
        return k

    if args.profile_steps:
        for _ in range(args.profile_steps):
            step()
        torch.cuda.synchronize()
        return None

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    uuid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid).replace("GPU-", "")
    sampler = ClockSampler(uuid)
    sampler.start()
    time.sleep(0.3)
    per = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    launches0 = _lib.kernel_launches()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for s in range(args.steps):
        step(per[s])
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = _lib.kernel_launches() - launches0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms_total = t_start.elapsed_time(t_end)
    det_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in per)
    des_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in per)
    if world > 1:
        t = torch.tensor([ms_total, det_ms, des_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total, det_ms, des_ms = t.tolist()
    ms_step = ms_total / args.steps
    # output sanity (not a parity test -- tests/ does that): every described
    # keypoint row is unit-norm, so a failed launch cannot pass as a fast one
    nrm = desc[:, : min(K, 4096)].double().norm(dim=-1)
    bad = int(((nrm - 1.0).abs() > 1e-5).sum())
    if bad:
        raise RuntimeError(f"describe produced {bad} non-unit descriptor rows")
    total_px = world * args.images * NR * NC  # all ranks' images
    value = total_px / 1e6 / (ms_step / 1e3)

    # ---- roofline (per launch on this rank's shard) ----
    peak, peak_kind = measured_peaks()
    n_kp = K * n
    bytes_detect = n * NR * NC + n_kp * 16  # image read + (row, col, value) out
    bytes_desc = n * NR * NC + n_kp * (16 + 128 * 4)  # image + keypoints in, fp32 rows out
    traffic, ncu_full = None, None
    tp = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        tr = tj.get("describe")
        if tr and int(tr.get("images", -1)) == n:
            traffic = tr["dram_bytes_per_launch"]
            ncu_full = tr.get("ncu_full")
    ach_des = bytes_desc / (des_ms / 1e3) / 1e9
    ach_det = bytes_detect / (det_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "kernel": "describe_f32_tile_kernel", "achieved": round(ach_des, 1), "peak": peak,
            "unit": "GB/s", "frac": round(ach_des / peak, 4), "traffic": traffic,
            "peak_source": peak_kind, "kernel_ms": round(des_ms, 4),
            "algorithmic_bytes_per_launch": bytes_desc,
            "note": "describe (float32 tile kernel + the float64 kernels for the border keypoints it queues) is "
                    "instruction-issue bound (issue below), not HBM-bound: bytes = 1 B/px + 16 B/kp in + "
                    "512 B/kp out; DRAM traffic from ncu equals the algorithmic bytes",
            "ncu": ncu_full}
    if ncu_full and ncu_full.get("warp_instructions"):
        # instruction roofline: warp instructions per launch (ncu, same launch) over this run's time,
        # against 4 issue slots per SM per clock at the sampled SM clock
        clk_hz = None  # filled after the clock sampler has run (below)
        roof["issue"] = {"warp_instructions_per_launch": ncu_full["warp_instructions"],
                         "source": ncu_full.get("source")}
    kernels = {"detect_u8_w8": {"ms": round(det_ms, 4), "GB/s": round(ach_det, 1),
                                "frac_hbm": round(ach_det / peak, 4), "bytes_per_launch": bytes_detect},
               "describe": {"ms": round(des_ms, 4), "GB/s": round(ach_des, 1),
                            "keypoints_per_s": round(n_kp / (des_ms / 1e3), 1)}}

    # detect alone, back to back (its inputs, 275 MB, exceed L2): the kernel's own roofline fraction,
    # without the write-back of the previous describe's dirty descriptor lines that it absorbs in the step
    iso = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(3):
        device.detect(dimg, SCALES, meta=False)
    iso[0].record(stream)
    n_iso = 20
    for _ in range(n_iso):
        device.detect(dimg, SCALES, meta=False)
    iso[1].record(stream)
    torch.cuda.synchronize()
    det_iso_ms = iso[0].elapsed_time(iso[1]) / n_iso
    if world > 1:
        t = torch.tensor([det_iso_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        det_iso_ms = t.item()
    ach_iso = bytes_detect / (det_iso_ms / 1e3) / 1e9
    kernels["detect_u8_w8"]["isolated"] = {"ms": round(det_iso_ms, 4), "GB/s": round(ach_iso, 1),
                                           "frac_hbm": round(ach_iso / peak, 4),
                                           "timing": f"CUDA events over {n_iso} back-to-back launches"}

    # the other configs' detector shapes, in isolation (random 8-bit rasters: the detector's work does
    # not depend on the content): bytes = 1 (3 for RGB) per pixel read + 16 per kept keypoint written
    if rank == 0 and not getattr(args, "no_match", False):
        kernels["detect_other_shapes"] = bench_detect_shapes(dev, peak)

    # ---- e2e through the public host API ----
    e2e = None
    if not args.no_e2e:
        pcfg = PipelineConfig(window_min=8, window_max=128)
        hin = torch.from_numpy(host).pin_memory()
        hout = alloc_host_features(n, NR, NC, pcfg)
        prep = BatchPreparer(NR, NC, pcfg, chunk=8)
        prep.run(hin, hout)
        torch.cuda.synchronize()
        e_steps = max(1, min(args.steps, 3))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            prep.run(hin, hout)
        torch.cuda.synchronize()
        e_ms = (time.perf_counter() - t0) * 1e3 / e_steps
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = t.item()
        d2h = n * (K * (4 + 4 + 8 + 128 * 4) + 4)
        e2e = {"value": round(total_px / 1e6 / (e_ms / 1e3), 2), "unit": "Mpixel/s", "ms_per_step": round(e_ms, 3),
               "steps": e_steps,
               "h2d_bytes_per_step": n * NR * NC * world, "d2h_bytes_per_step": d2h * world,
               "api": "paper_2405_08578_b200.pipeline.BatchPreparer.run (pinned host in/out, 3-stream pipeline)"}

    cpu = None
    with_cpu = rank == 0 and world == 1 and not args.no_cpu
    if with_cpu:
        cpu = cpu_baseline(steps=1, warmup=0)
    # the float64 kernels (PS_DESCRIBE_PRECISE; the path of float64-output calls such as the
    # reference-facing describe_features): same batch, CUDA events, with the FP64-pipe peak probe
    pe = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    device.describe_into(dimg, kp, cfg, desc, scale_set=kp.scale_set, policy="precise")
    pe[0].record(stream)
    for _ in range(3):
        device.describe_into(dimg, kp, cfg, desc, scale_set=kp.scale_set, policy="precise")
    pe[1].record(stream)
    torch.cuda.synchronize()
    fp64 = fp64_probe(dev)
    kernels["describe_precise_f64"] = {
        "ms": round(pe[0].elapsed_time(pe[1]) / 3, 4), "fp64_peak_tflops_measured": fp64["tflops"],
        "probe": fp64["how"],
        "note": "float64 kernels (describe_pair_kernel + describe_kernel), ~1e-14 from the reference; "
                "the headline float32 kernel is ~1e-7 (P2 bar 1e-4)"}

    if "issue" in roof:
        mhz = (clocks or {}).get("sm_mhz") or 1965.0
        peak_issue = 148 * 4 * mhz * 1e6  # warp instructions per second, all SMs
        ach = roof["issue"]["warp_instructions_per_launch"] / (des_ms / 1e3)
        roof["issue"].update({"achieved_per_s": round(ach, 1), "peak_per_s": round(peak_issue, 1),
                              "frac": round(ach / peak_issue, 4), "sm_mhz": mhz,
                              "note": "4 warp-instruction issue slots per SM per clock (148 SMs)"})

    latency = None
    if not args.no_stitch:
        latency = bench_c1_latency(args, rank, dev, with_cpu=with_cpu)

    stitch = None
    if not args.no_stitch:
        stitch = bench_c3_stitch(args, world, rank, dev, with_cpu=with_cpu)

    composite = None
    if not args.no_composite:
        composite = bench_c3_composite(args, rank, dev, with_cpu=(not args.no_cpu and world == 1))

    ransac_k4 = None
    if not args.no_pairs:
        ransac_k4 = bench_ransac(args, rank, dev, with_cpu=(not args.no_cpu and world == 1))

    pairs5 = None
    if not args.no_pairs:
        pairs5 = bench_c5_pairs(args, world, rank, dev, with_cpu=with_cpu)

    matching = None
    if not args.no_match:
        del desc, imgs, dimg
        torch.cuda.empty_cache()
        matching = bench_c4_matching(args, world, rank, dev, with_cpu=(not args.no_cpu and world == 1))
        torch.cuda.empty_cache()
        matching_dense = bench_c4_dense(args, rank, dev)
    else:
        matching_dense = None

    if rank == 0:
        out = {
            "metric": "Mpixel/s LP-SIFT detect+describe", "value": round(value, 2), "unit": "Mpixel/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8/f32",
            "data": "synthetic (seeded noise+shapes generator, paper_2405_08578_b200/scenes.py)",
            "config": {"workload": WORKLOAD, "images": args.images, "image_hw": [NR, NC], "scales": list(SCALES),
                       "keypoints_per_image": K, "descriptor": "float32 128-d", "l2": "inputs larger than L2",
                       "parallelism": f"{world} rank(s) x one 64-image C2 batch each (weak scaling, no collective)"},
            "roofline": roof, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e, "latency_c1": latency,
            "matching_c4": matching, "matching_c4_dense": matching_dense,
            "stitch_c3": stitch, "composite_c3": composite, "pairs_c5": pairs5, "ransac_k4": ransac_k4,
            "gpu_launches": int(launches), "clocks": clocks,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return None


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_baseline(steps=max(args.steps, 1), warmup=max(args.warmup, 0) and 1)
    out = {"metric": "Mpixel/s LP-SIFT detect+describe", "value": round(cb["value"], 4), "unit": "Mpixel/s",
           "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded noise+shapes generator)",
           "config": {"workload": WORKLOAD, "images": args.images, "image_hw": [NR, NC], "scales": list(SCALES)},
           "cpu_baseline": cb,
           "e2e": {"value": round(cb["value"], 4), "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def _spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch this script as N
    NCCL ranks on this node (torch.distributed.run, 127.0.0.1)."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        sys.exit(_spawn_ranks(args))
    if world and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
