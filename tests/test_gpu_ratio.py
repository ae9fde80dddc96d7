"""The extra "ratio_test" matching strategy (north star: Lowe ratio 0.8; not
in the reference) against its own numpy oracle
(oracle/lpsift_oracle.py ``match(..., strategy="ratio_test")``), bit-exact:
same (ref1, ref2) set and order, delta bits equal."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import lpsift_oracle as O  # noqa: E402
from paper_2405_08578_b200 import device, matcher as Mt, records as R, scenes  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def check(A, B, ratio=0.8):
    r1, r2, dl = device.match(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), ratio, "ratio_test")
    w1, w2, wd = O.match(A.astype(np.float64), B.astype(np.float64), ratio, "ratio_test")
    assert np.array_equal(r1.cpu().numpy(), w1) and np.array_equal(r2.cpu().numpy(), w2)
    assert np.array_equal(dl.cpu().numpy(), wd)
    return len(w1)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_ratio_random_with_ties_and_near_copies(dtype):
    rng = np.random.default_rng(31)
    A = rng.random((700, 128)).astype(dtype)
    B = rng.random((650, 128)).astype(dtype)
    B[:300] = (A[:300] + rng.normal(0, 0.02, (300, 128))).astype(dtype)
    B[300:304] = A[0]  # duplicated best column: d2 == d1 -> rejected
    A[5] = A[6]
    for ratio in (0.8, 0.5, 1.0):
        n = check(A, B, ratio)
        assert n > 0


def test_ratio_edge_cases():
    rng = np.random.default_rng(2)
    A = rng.random((17, 128)).astype(np.float32)
    assert check(A, A[:1]) == 17  # one column: d2 = inf, every row kept
    e = torch.zeros((0, 128), device="cuda")
    r1, _, _ = device.match(e, torch.from_numpy(A).cuda(), 0.8, "ratio_test")
    assert r1.numel() == 0
    with pytest.raises(Exception):
        device.match(torch.from_numpy(A).cuda(), torch.from_numpy(A).cuda(), 1.5, "ratio_test")


def test_ratio_on_c1_pair_and_drop_in():
    a, b = scenes.config1_pair(0)
    cfg = R.DescriptorConfig(0.0625, 4, 64, True)
    ds, feats = [], []
    for im in (a, b):
        t = torch.from_numpy(im).cuda()
        kp = device.detect(t, (16, 32, 64))
        ds.append(device.describe(t, kp, cfg)[0].cpu().numpy())
        h = kp.image(0)
        feats.append([R.FeaturePoint(int(r), int(c), 16, "max", 0, 0.0) for r, c in zip(h["row"], h["col"])])
    n = check(ds[0], ds[1])
    assert n > 100
    pairs = Mt.match_features(R.DescribedFeatures("a", feats[0], ds[0]), R.DescribedFeatures("b", feats[1], ds[1]),
                              R.MatcherConfig(strategy="ratio_test", ratio=0.8))
    assert len(pairs) == n
