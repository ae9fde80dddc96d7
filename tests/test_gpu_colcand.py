"""Column candidates (csrc/match_tc.cu ColCand): the tensor-core matcher decides
the mutual test from pass 1's exact distances below delta_s and skips the
column pass when that list is complete.  Its result must equal the float64
CUDA-core path (pinned to the oracle / reference fixtures in test_gpu_parity.py
P3) bit for bit -- on data where the single pass is taken (``passes`` == 1),
on columns contested by several rows (closest wins, lowest row index at
exactly equal distances), and on clustered data where it must fall back to two
passes.  The reference rule: matcher.py:74-79 (argmin rows, argmin columns,
mutual, distance < delta_s).
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2405_08578_b200 import device  # noqa: E402


def _unit(x):
    return x / np.maximum(np.linalg.norm(x, axis=1, keepdims=True), 1e-12)


def _same(a, b):
    for x, y in zip(a, b):
        assert torch.equal(x.cpu(), y.cpu())


def _both(A, B, delta_s=0.35):
    t = device.match(A, B, delta_s, path="tensor")
    passes = device.match_stats()["passes"]
    e = device.match(A, B, delta_s, path="exact")
    _same(t, e)
    r1, r2, dl, cnt = device.match_batch_async([A, B], [(0, 1), (1, 0)], delta_s)
    torch.cuda.synchronize()
    m = int(cnt[0].item())
    assert m == int(e[0].shape[0])
    _same((r1[0, :m].long(), r2[0, :m].long(), dl[0, :m]), (e[0].long(), e[1].long(), e[2]))
    e2 = device.match(B, A, delta_s, path="exact")
    m2 = int(cnt[1].item())
    assert m2 == int(e2[0].shape[0])
    _same((r1[1, :m2].long(), r2[1, :m2].long(), dl[1, :m2]), (e2[0].long(), e2[1].long(), e2[2]))
    return int(e[0].shape[0]), passes


def test_single_pass_on_distinct_rows():
    rng = np.random.default_rng(5)
    a = _unit(rng.random((6000, 128)))
    b = _unit(rng.random((7000, 128)))
    b[:3000] = _unit(a[rng.permutation(6000)[:3000]] + 0.01 * rng.standard_normal((3000, 128)))
    A, B = torch.from_numpy(a).float().cuda(), torch.from_numpy(b).float().cuda()
    m, passes = _both(A, B)
    assert m >= 2900 and passes == 1


def test_contested_columns_and_equal_distances():
    rng = np.random.default_rng(6)
    b = _unit(rng.random((4096, 128)))
    a = _unit(rng.random((5000, 128)))
    # rows 0..999: two copies of b_j at different distances (the closer one wins column j)
    perm = rng.permutation(4096)
    j = perm[:500]
    a[0:1000:2] = b[j] + 0.02 * rng.standard_normal((500, 128))
    a[1:1000:2] = b[j] + 0.005 * rng.standard_normal((500, 128))
    A = torch.from_numpy(a).float().cuda()
    B = torch.from_numpy(b).float().cuda()
    # rows 2000..2199: pairs of distinct rows at exactly the same float64 distance from b_k
    # (b_k +- e with e representable: the squared differences are bitwise equal): the lower index wins
    k = perm[500:600]
    Bf = B[torch.from_numpy(k).cuda()].clone()
    e = torch.zeros(128, device="cuda")
    e[3] = 2.0 ** -6
    e[77] = 2.0 ** -7
    Bq = (Bf * 1024).round() / 1024  # coarse grid: b +- e exact in float32
    B[torch.from_numpy(k).cuda()] = Bq
    A[2000:2200:2] = Bq + e
    A[2001:2200:2] = Bq - e
    m, passes = _both(A, B)
    assert m >= 500 and passes == 1
    r1, r2, _ = device.match(A, B, 0.35, path="tensor")
    got = dict(zip(r2.tolist(), r1.tolist()))
    for t, kk in enumerate(k.tolist()):
        assert got.get(kk) == 2000 + 2 * t  # the lower of the two equidistant rows
    for t, jj in enumerate(j.tolist()):
        assert got.get(jj) == 2 * t + 1  # the closer copy


def test_clustered_rows_fall_back_to_two_passes():
    rng = np.random.default_rng(7)
    centres = _unit(rng.random((200, 128)))
    a = _unit(centres[rng.integers(0, 200, 5000)] + 0.02 * rng.standard_normal((5000, 128)))
    b = _unit(centres[rng.integers(0, 200, 5000)] + 0.02 * rng.standard_normal((5000, 128)))
    A, B = torch.from_numpy(a).float().cuda(), torch.from_numpy(b).float().cuda()
    # ~25 columns below delta_s per row, spread well beyond the certification margin: the top-4
    # cannot hold a row's column candidates, so the column pass must run
    m, passes = _both(A, B)
    assert passes == 2 and m > 0


def test_near_tied_clusters_are_enumerated():
    rng = np.random.default_rng(9)
    centres = _unit(rng.random((40, 128)))
    a = _unit(centres[rng.integers(0, 40, 5000)] + 0.004 * rng.standard_normal((5000, 128)))
    b = _unit(centres[rng.integers(0, 40, 5000)] + 0.004 * rng.standard_normal((5000, 128)))
    A, B = torch.from_numpy(a).float().cuda(), torch.from_numpy(b).float().cuda()
    m, _ = _both(A, B)  # hundreds of near-tied columns per row: overflow rows, enumerated up to delta_s
    assert m > 0


def test_float64_descriptors_and_threshold_edge():
    rng = np.random.default_rng(8)
    a = _unit(rng.random((3000, 128)))
    b = _unit(a[rng.permutation(3000)] + 0.02 * rng.standard_normal((3000, 128)))
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    m, _ = _both(A, B)
    assert m > 2500
    # a threshold inside the distance distribution: pairs just above / below delta_s
    d = np.sort(np.linalg.norm(a[:, None, :] - b[None, :64, :], axis=2).min(axis=0))
    _both(A, B, float(d[32]))
    _both(A, B, float(np.nextafter(d[32], 0.0)))
