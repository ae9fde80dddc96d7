"""Batched pair matching (ps_match_batch_async) against the per-pair matcher.

``device.match`` is pinned to the oracle / reference fixtures elsewhere
(test_gpu_parity.py P3, test_gpu_pairs.py, test_gpu_c4.py); the batch runs
the same kernel bodies per pair, so every pair's (ref1, ref2, delta) list and
count must be bit-identical to ``device.match`` on the same two sets --
including sets shared by several pairs, a set matched with itself, duplicate
rows, empty sets and float64 descriptors.  The C3 table (9 images, 36 pairs,
every image in 8 pairs) is checked through the engine the bench times.
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2405_08578_b200 import device, scenes  # noqa: E402
from paper_2405_08578_b200.pipeline import PipelineConfig  # noqa: E402


def _unit_rows(rng, n, dup_every=0, dtype=torch.float32):
    x = rng.standard_normal((n, 128))
    x = np.abs(x) * (rng.random((n, 128)) < 0.4)  # sparse, non-negative like SIFT rows
    x /= np.maximum(np.linalg.norm(x, axis=1, keepdims=True), 1e-12)
    if dup_every:
        x[::dup_every] = x[0]  # a cluster of bit-identical rows (saturated regions)
    return torch.from_numpy(x).to(dtype).cuda()


def _perturbed(rng, base, sigma, n_extra):
    x = base.double().cpu().numpy()
    y = x[rng.permutation(x.shape[0])] + sigma * rng.standard_normal(x.shape)
    y = np.vstack([y, np.abs(rng.standard_normal((n_extra, 128)))])
    y = np.abs(y)
    y /= np.maximum(np.linalg.norm(y, axis=1, keepdims=True), 1e-12)
    return torch.from_numpy(y).to(base.dtype).cuda()


def _check(sets, pairs, delta_s=0.35):
    r1, r2, dl, cnt = device.match_batch_async(sets, pairs, delta_s)
    torch.cuda.synchronize()
    cnt = cnt.cpu().numpy()
    for q, (a, b) in enumerate(pairs):
        e1, e2, ed = device.match(sets[a], sets[b], delta_s, path="tensor") if min(
            sets[a].shape[0], sets[b].shape[0]) else (torch.zeros(0), torch.zeros(0), torch.zeros(0))
        m = int(e1.shape[0])
        assert int(cnt[q]) == m, (q, a, b, int(cnt[q]), m)
        assert torch.equal(r1[q, :m].cpu(), e1.cpu().to(torch.int32)), (q, a, b)
        assert torch.equal(r2[q, :m].cpu(), e2.cpu().to(torch.int32)), (q, a, b)
        assert torch.equal(dl[q, :m].cpu(), ed.cpu().to(torch.float64)), (q, a, b)
    return cnt


def test_batch_equals_per_pair_shared_sets():
    rng = np.random.default_rng(11)
    base = _unit_rows(rng, 3000, dup_every=97)
    sets = [base, _perturbed(rng, base, 0.01, 500), _perturbed(rng, base, 0.03, 0),
            _unit_rows(rng, 1200), _perturbed(rng, base[:700], 0.005, 60)]
    pairs = [(0, 1), (0, 2), (1, 2), (2, 0), (3, 0), (0, 3), (4, 1), (1, 4), (2, 2), (3, 4)]
    cnt = _check(sets, pairs)
    assert cnt[0] > 1000 and cnt[8] > 0  # real matches, including the self pair


def test_batch_sizes_and_edge_cases():
    rng = np.random.default_rng(5)
    a = _unit_rows(rng, 1)
    b = _unit_rows(rng, 300)
    c = _unit_rows(rng, 129)  # one past a row block
    d = _unit_rows(rng, 256 * 3 + 1, dup_every=2)  # half the rows identical
    e = torch.zeros((0, 128), dtype=torch.float32, device="cuda")
    f = _unit_rows(rng, 3000)
    for k in range(0, 3000, 37):  # runs of consecutive identical rows (flat regions), some chunk-straddling
        f[k:k + 1 + k % 23] = f[k]
    f[1500:1900] = f[1499]
    sets = [a, b, c, d, e, f]
    pairs = [(0, 1), (1, 0), (1, 2), (2, 3), (3, 2), (3, 3), (0, 0), (4, 1), (1, 4), (5, 3), (3, 5), (5, 5)]
    cnt = _check(sets, pairs, delta_s=10.0)  # every mutual pair accepted
    assert cnt[7] == 0 and cnt[8] == 0 and cnt[6] == 1


def test_batch_float64_sets():
    rng = np.random.default_rng(8)
    base = _unit_rows(rng, 1500, dtype=torch.float64)
    sets = [base, _perturbed(rng, base, 0.02, 100), _perturbed(rng, base, 0.02, 0)]
    _check(sets, [(0, 1), (1, 2), (2, 0)])


def test_batch_many_pairs_chunked():
    """More pairs than one call takes (BATCH_MAX_PAIRS): chunked launches."""
    rng = np.random.default_rng(3)
    sets = [_unit_rows(rng, 200 + 7 * k) for k in range(24)]
    pairs = [(i, j) for i in range(24) for j in range(24) if i != j][: device.BATCH_MAX_PAIRS + 40]
    r1, r2, dl, cnt = device.match_batch_async(sets, pairs, 1.5)
    torch.cuda.synchronize()
    for q in (0, 17, device.BATCH_MAX_PAIRS - 1, device.BATCH_MAX_PAIRS, len(pairs) - 1):
        a, b = pairs[q]
        e1, e2, ed = device.match(sets[a], sets[b], 1.5, path="tensor")
        m = int(e1.shape[0])
        assert int(cnt[q]) == m
        assert torch.equal(r1[q, :m], e1.to(torch.int32)) and torch.equal(r2[q, :m], e2.to(torch.int32))
        assert torch.equal(dl[q, :m], ed)


def test_batch_c3_table_equals_per_pair():
    """C3 (9 x 2688x1600 crops, 36 pairs): the batch on the images'
    descriptor sets equals device.match pair by pair, and the engine's
    table (batched) equals the per-pair-launch engine's."""
    from paper_2405_08578_b200 import mosaic

    imgs, _ = scenes.config3_images()
    cfg = PipelineConfig()
    eng = mosaic.GpuEngine(cfg)
    rows, cols, desc, count = eng.prepare(imgs)
    n = count.cpu().tolist()
    sets = [desc[k, : n[k]] for k in range(len(imgs))]
    pairs = [(a, b) for a in range(len(imgs)) for b in range(a + 1, len(imgs))]
    cnt = _check(sets, pairs)
    assert cnt.sum() > 0
    control, _ = scenes.config3_images(0, rot_deg=0.0, scale_range=(1.0, 1.0), noise=0.0)
    for images, min_registered in ((imgs, 0), (control, 15)):
        t_batch = mosaic.build_pairwise_table(images, cfg, engine=eng)
        eng2 = mosaic.GpuEngine(cfg)
        eng2.batch_match = False
        t_pair = mosaic.build_pairwise_table(images, cfg, engine=eng2)
        assert t_batch.entries.keys() == t_pair.entries.keys()
        assert len(t_batch.entries) >= 2 * min_registered
        for k, v in t_batch.entries.items():
            w = t_pair.entries[k]
            assert v.inlier_count == w.inlier_count and v.transform == w.transform


def test_batch_graph_replay_c5_pairs():
    """C5-style disjoint pairs (RGB, homography warp) through the graph
    engine: replays equal the eager batched phase and the per-pair path."""
    from paper_2405_08578_b200 import mosaic

    cfg = PipelineConfig(window_min=16, window_max=64)
    pairs = [scenes.config5_pair(k) for k in range(6)]
    batch = torch.from_numpy(np.stack([im for a, b, _ in pairs for im in (a, b)])).cuda()
    g = device.as_device_images(batch, rgb=True)
    eng = mosaic.GraphEngine(cfg)
    rows, cols, desc, count = eng.prepare_device(g)
    n = count.cpu().tolist()
    items = [(rows[2 * k], cols[2 * k], desc[2 * k], n[2 * k], rows[2 * k + 1], cols[2 * k + 1], desc[2 * k + 1],
              n[2 * k + 1], 1000 + k) for k in range(len(pairs))]
    first = eng.register_many(items)  # eager + capture
    again = eng.register_many(items)  # replay
    ref = [eng.register(*it) for it in items]
    assert first == again == ref


def test_batch_graph_replay_with_device_counts_that_change():
    """Items carrying device keypoint counts (build_pairwise_table's form):
    the pair graph is keyed on slot capacities, so frames whose counts differ
    replay the SAME graph (no re-capture) and still equal the per-pair path
    on the truncated sets -- including a pair whose count falls below
    min_inliers (RegistrationError decided on the device)."""
    from paper_2405_08578_b200 import mosaic

    cfg = PipelineConfig(window_min=16, window_max=64)
    pairs = [scenes.config5_pair(k) for k in range(4)]
    batch = torch.from_numpy(np.stack([im for a, b, _ in pairs for im in (a, b)])).cuda()
    g = device.as_device_images(batch, rgb=True)
    eng = mosaic.GraphEngine(cfg)
    rows, cols, desc, count = eng.prepare_device(g)
    full = count.cpu().tolist()
    live = torch.zeros(len(full), dtype=torch.int32, device=count.device)  # the counts the graph reads
    items = [(rows[2 * k], cols[2 * k], desc[2 * k], full[2 * k], rows[2 * k + 1], cols[2 * k + 1],
              desc[2 * k + 1], full[2 * k + 1], 2000 + k, live[2 * k:2 * k + 1], live[2 * k + 1:2 * k + 2])
             for k in range(len(pairs))]
    rng = np.random.default_rng(4)
    for frame in range(3):
        n = [int(c) if frame == 0 else int(rng.integers(c // 3, c + 1)) for c in full]
        if frame == 2:
            n[0] = 5  # below min_inliers: no registration
        live.copy_(torch.tensor(n, dtype=torch.int32))
        got = eng.register_many(items)
        assert len(eng._pair_graphs) == 1  # captured once, replayed for every frame
        want = [eng.register(*it[:3], n[2 * k], *it[4:7], n[2 * k + 1], it[8]) for k, it in enumerate(items)]
        assert got == want, frame
        if frame == 2:
            assert got[0][0] is False


def test_register_batch_equals_per_pair_ransac():
    """ps_register_batch_async vs pair_points_dev + ransac_async_dev per pair:
    rigid pairs with outliers, a pair whose count is below min_inliers, a
    skipped pair; identical result blocks (model, rms, status words, mask)."""
    rng = np.random.default_rng(21)
    P, S, iters, tol, min_in = 5, 600, 500, 3.0, 4
    kp = []  # per pair: (row1, col1, row2, col2) int32 device arrays
    r1 = torch.zeros((P, S), dtype=torch.int32)
    r2 = torch.zeros((P, S), dtype=torch.int32)
    counts = torch.tensor([S, 400, 3, 250, S], dtype=torch.int64)
    for q in range(P):
        n1, n2 = 900, 800
        rows1, cols1 = rng.integers(0, 1600, n1), rng.integers(0, 2688, n1)
        th, tx, ty = rng.uniform(-0.1, 0.1), rng.uniform(-300, 300), rng.uniform(-200, 200)
        # image-2 keypoints: a rigid map of image-1 keypoints (rounded) plus clutter
        idx = rng.permutation(n1)[:n2]
        x2 = np.cos(th) * cols1[idx] - np.sin(th) * rows1[idx] + tx
        y2 = np.sin(th) * cols1[idx] + np.cos(th) * rows1[idx] + ty
        out = rng.random(n2) < 0.3
        x2 = np.where(out, rng.integers(0, 2688, n2), np.rint(x2))
        y2 = np.where(out, rng.integers(0, 1600, n2), np.rint(y2))
        kp.append(tuple(torch.from_numpy(np.asarray(a, dtype=np.int32)).cuda() for a in (rows1, cols1, y2, x2)))
        m = int(counts[q])
        sel = rng.permutation(n2)[:m]
        r1[q, :m] = torch.from_numpy(idx[sel].astype(np.int32))
        r2[q, :m] = torch.from_numpy(sel.astype(np.int32))
    r1, r2, counts = r1.cuda(), r2.cuda(), counts.cuda()
    width = 8 + (S + 7) // 8
    got = torch.zeros((P, width), dtype=torch.float64, device="cuda")
    jobs = [(kp[q][0], kp[q][1], kp[q][2], kp[q][3], S, 100 + q) if q != 4 else None for q in range(P)]
    device.register_batch_async(jobs, r1, r2, counts, iters, tol, min_in, got)
    want = torch.zeros((P, width), dtype=torch.float64, device="cuda")
    for q in range(4):
        src, dst = device.pair_points_dev(r1[q], r2[q], counts[q:q + 1], *kp[q])
        device.ransac_async_dev(src, dst, counts[q:q + 1], S, iters, tol, min_in, 100 + q, want[q])
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.uint8), want.view(torch.uint8))
    info = got[:, 4:8].contiguous().view(torch.int64).cpu().numpy()
    assert info[0, 0] == 0 and info[2, 0] != 0 and info[0, 2] > 300  # registered / too few pairs
    assert not got[4].any()  # skipped pair untouched
