"""GPU parity: the CUDA path (through the C-ABI) against the reference's own
outputs (tests/golden, produced by tests/golden/make_golden.py) and the
pinned CPU oracle (oracle/lpsift_oracle.py).

Bars:
  P1 keypoints: row/col/scale/polarity/window exact and in order, value bit-exact;
  P2 descriptors: max|gpu - ref| / ||ref||_2 <= 1e-4 per keypoint (float64 path
     is expected <= 1e-12 away; the bar is the contract's);
  P3 matches on identical descriptors: (ref1, ref2) and delta bit-exact;
  P4 RANSAC: inlier list, consensus and success exact; transform within
     1e-3 px at the image corners;
  P5 end to end: every match-set difference classified as a near-tie under the
     measured descriptor perturbation (tests/match_diff.py), none unexplained.
"""

import json
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import lpsift_oracle as O  # noqa: E402
from paper_2405_08578_b200 import descriptor as Dsc  # noqa: E402
from paper_2405_08578_b200 import detector as Det  # noqa: E402
from paper_2405_08578_b200 import device, records as R, scenes  # noqa: E402
from paper_2405_08578_b200 import matcher as Mt  # noqa: E402
from paper_2405_08578_b200 import registration as Rg  # noqa: E402
from paper_2405_08578_b200.errors import DegenerateSampleError, RegistrationError  # noqa: E402
from match_diff import classify, ref_match_with_gaps  # noqa: E402

P2_TOL = 1e-4
KP = ("row", "col", "scale", "pol", "window", "value")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def kp_arrays(feats):
    return dict(row=np.array([f.row for f in feats]), col=np.array([f.col for f in feats]),
                scale=np.array([f.scale for f in feats]), pol=np.array([f.polarity == "min" for f in feats], np.int8),
                window=np.array([f.window_index for f in feats]), value=np.array([f.value for f in feats]))


def assert_kp_equal(got: dict, want, label=""):
    for f in KP:
        g, w = np.asarray(got[f]), np.asarray(want[f])
        assert g.shape == w.shape, (label, f, g.shape, w.shape)
        assert np.array_equal(g.astype(w.dtype) if f != "value" else g, w), (label, f)


# ---------------------------------------------------------------------------
# P1 -- detector
# ---------------------------------------------------------------------------

def test_detector_matches_reference_fixtures(golden):
    g = golden("detector.npz")
    meta = json.loads(str(g["meta"]))
    for m in meta:
        lab = m["label"]
        px = g[f"{lab}__pixels"]
        want = {f: g[f"{lab}__{f}"] for f in KP}
        # (a) drop-in path: RampedImage from apply_linear_ramp (fused ramp; u8 key path when integral)
        img = R.apply_linear_ramp(R.IntensityImage(px), m["alpha"])
        feats = Det.detect_features(img, R.ScaleSet(tuple(m["scales"])), dedupe=m["dedupe"])
        assert_kp_equal(kp_arrays(feats), want, lab + "/fused")
        # (b) a materialised float64 RampedImage (reference-style object)
        P = O.ramp(px.astype(np.float64), m["alpha"])
        img2 = R.RampedImage(pixels=P, alpha=m["alpha"], source_id="x")
        feats2 = Det.detect_features(img2, R.ScaleSet(tuple(m["scales"])), dedupe=m["dedupe"])
        assert_kp_equal(kp_arrays(feats2), want, lab + "/f64")


@pytest.mark.parametrize("shape,scales", [
    ((768, 1024), (16, 32, 64)), ((1600, 2688), (8, 16, 32, 64, 128)), ((1600, 2688), (32, 64, 128)),
    ((1080, 1920), (16, 32, 64)), ((1037, 1501), (8, 16, 32)), ((300, 333), (8, 12, 24)),
    ((513, 777), (32, 40)), ((256, 256), (8, 9, 128)),
])
def test_detector_u8_matches_oracle_full_size(shape, scales):
    img = scenes.scene(shape[0], shape[1], seed=shape[0] + shape[1])
    alpha = O.default_alpha(*shape)
    want = O.detect(O.ramp(img.astype(np.float64), alpha), scales)
    kp = device.detect(torch.from_numpy(img).cuda(), scales, alpha=alpha)
    h = kp.image(0)
    h["pol"] = h.pop("polarity")
    assert_kp_equal(h, want, str(shape))


def test_detector_batch_and_no_meta_fast_path():
    imgs = np.stack([scenes.scene(200, 352, s) for s in range(5)])
    alpha = O.default_alpha(200, 352)
    kp = device.detect(torch.from_numpy(imgs).cuda(), (8, 16, 32), alpha=alpha, meta=False)
    assert kp.count.cpu().tolist() == [2 * 25 * 44] * 5
    for b in range(5):
        want = O.detect(O.ramp(imgs[b].astype(np.float64), alpha), (8, 16, 32))
        h = kp.image(b)
        assert np.array_equal(h["row"], want["row"]) and np.array_equal(h["col"], want["col"])
        assert np.array_equal(h["value"], want["value"])


def test_detector_tie_heavy_u8_random():
    rng = np.random.default_rng(5)
    for t in range(50):
        px = (rng.integers(0, 3, size=(64, 64)) * 100).astype(np.uint8)
        alpha = O.default_alpha(64, 64)
        for scales in [(8, 16, 32), (32, 40) if t % 2 else (16, 24)]:
            want = O.detect(O.ramp(px.astype(np.float64), alpha), scales)
            feats = Det.detect_features(R.apply_linear_ramp(R.IntensityImage(px), alpha), R.ScaleSet(scales))
            assert_kp_equal(kp_arrays(feats), want, f"tie{t}")


def test_detector_tiny_alpha_uses_exact_float_path():
    rng = np.random.default_rng(9)
    px = rng.integers(0, 2, size=(96, 80)).astype(np.uint8)
    for alpha in (1e-15, 1e-3):  # key rule invalid: float64 comparison on P
        want = O.detect(O.ramp(px.astype(np.float64), alpha), (8, 16))
        feats = Det.detect_features(R.apply_linear_ramp(R.IntensityImage(px), alpha), R.ScaleSet((8, 16)))
        assert_kp_equal(kp_arrays(feats), want, str(alpha))


# ---------------------------------------------------------------------------
# P2 -- descriptor
# ---------------------------------------------------------------------------

def test_descriptor_matches_reference_fixtures(golden):
    g = golden("descriptor.npz")
    worst = 0.0
    for i in range(len(g["row"])):
        iid = int(g["img_id"][i])
        px = g[f"img{iid}"]
        if f"alpha{iid}" in g.files:
            img = R.apply_linear_ramp(R.IntensityImage(px), float(g[f"alpha{iid}"]))
        else:
            img = R.RampedImage(pixels=px.astype(np.float64), alpha=1e-9, source_id="t")
        cfg = R.DescriptorConfig(float(g["beta0"][i]), int(g["d"][i]), int(g["l_max"][i]), bool(g["orient"][i]))
        fp = R.FeaturePoint(int(g["row"][i]), int(g["col"][i]), int(g["scale"][i]), "max", 0, 0.0)
        got = Dsc.compute_descriptor(img, fp, cfg).values
        ref = g["desc"][i]
        nrm = max(np.linalg.norm(ref), 1e-300)
        err = float(np.max(np.abs(got - ref))) / nrm if np.any(ref) else float(np.max(np.abs(got)))
        worst = max(worst, err)
    assert worst <= P2_TOL, worst


def test_descriptor_full_c2_image_sampled_against_oracle():
    img = scenes.scene(1600, 2688, 0)
    alpha = O.default_alpha(1600, 2688)
    cfg = R.DescriptorConfig(0.0625, 4, 128, True)
    t = torch.from_numpy(img).cuda()
    kp = device.detect(t, (8, 16, 32, 64, 128), alpha=alpha, meta=False)
    d32, d64 = device.describe(t, kp, cfg, out64=True)
    d32_only = device.describe(t, kp, cfg)  # float32-only output path (float32 normalisation)
    assert int(kp.count[0]) == 134400
    P = O.ramp(img.astype(np.float64), alpha)
    h = kp.image(0)
    rng = np.random.default_rng(0)
    idx = rng.choice(134400, 400, replace=False)
    worst = 0.0
    for k in idx:
        want = O.describe_one(P, int(h["row"][k]), int(h["col"][k]), 8, 0.0625, 4, 128, True)
        got = d64[0, k].cpu().numpy()
        worst = max(worst, float(np.max(np.abs(got - want)) / max(np.linalg.norm(want), 1e-300)))
        g32 = d32_only[0, k].double().cpu().numpy()
        worst = max(worst, float(np.max(np.abs(g32 - want)) / max(np.linalg.norm(want), 1e-300)))
        assert np.array_equal(d32[0, k].cpu().numpy(), got.astype(np.float32))
    assert worst <= P2_TOL, worst


def test_descriptor_saturated_clusters_bit_identical_and_deterministic():
    img = scenes.scene(768, 1024, 1)
    t = torch.from_numpy(img).cuda()
    cfg = R.DescriptorConfig(0.0625, 4, 64, True)
    kp = device.detect(t, (16, 32, 64), meta=False)
    a = device.describe(t, kp, cfg)
    b = device.describe(t, kp, cfg)
    assert torch.equal(a, b)
    uniq = torch.unique(a[0], dim=0).shape[0]
    assert uniq < a.shape[1]  # flat regions produce identical (saturated) rows
    # rows bit-identical in the oracle are bit-identical on the GPU
    d64 = device.describe(t, kp, cfg, out64=True, out32=False)[0].cpu().numpy()
    P = O.ramp(img.astype(np.float64), O.default_alpha(*img.shape))
    h = kp.image(0)
    idx = np.random.default_rng(3).choice(len(h["row"]), 1500, replace=False)
    groups = {}
    for k in idx:
        ref = O.describe_one(P, int(h["row"][k]), int(h["col"][k]), 16, 0.0625, 4, 64, True)
        groups.setdefault(ref.tobytes(), []).append(int(k))
    multi = [g for g in groups.values() if len(g) > 1]
    assert multi
    for g in multi:
        assert all(np.array_equal(d64[g[0]], d64[k]) for k in g[1:]), g


def test_descriptor_properties():
    rng = np.random.default_rng(7)
    px = rng.uniform(0, 255, size=(80, 80))
    img = R.RampedImage(pixels=px, alpha=1e-9, source_id="t")
    v = Dsc.compute_descriptor(img, R.FeaturePoint(40, 40, 32, "max", 0, 0.0), R.DescriptorConfig(l_max=32))
    assert np.all(v.values >= 0) and abs(np.linalg.norm(v.values) - 1) < 1e-9
    flat = R.RampedImage(pixels=np.full((64, 64), 9.0), alpha=1e-9, source_id="t")
    for on in (True, False):
        z = Dsc.compute_descriptor(flat, R.FeaturePoint(32, 32, 32, "max", 0, 0.0),
                                   R.DescriptorConfig(l_max=32, orientation_normalize=on))
        assert np.all(z.values == 0.0)
    grad = R.RampedImage(pixels=np.arange(64)[None, :] * 3.0 + np.zeros((64, 64)), alpha=1e-9, source_id="t")
    for on in (True, False):
        u = Dsc.compute_descriptor(grad, R.FeaturePoint(32, 32, 32, "max", 0, 0.0),
                                   R.DescriptorConfig(l_max=32, orientation_normalize=on)).values
        nz = u[u > 0]
        assert len(nz) == 16 and np.allclose(nz, 0.25, atol=1e-9)
    d = Dsc.describe_features(img, [], R.DescriptorConfig(l_max=32))
    assert d.descriptors.shape == (0, 128)


# ---------------------------------------------------------------------------
# P3 -- matcher
# ---------------------------------------------------------------------------

def described(desc):
    feats = [R.FeaturePoint(i, 0, 16, "max", 0, 0.0) for i in range(len(desc))]
    return R.DescribedFeatures("m", feats, np.asarray(desc))


def test_matcher_matches_reference_fixtures(golden):
    g = golden("matcher.npz")
    for m in json.loads(str(g["meta"])):
        A, B = g[f"{m['label']}__A"], g[f"{m['label']}__B"]
        for arr_a, arr_b in ((A, B), (A.astype(np.float64), B.astype(np.float64))):
            pairs = Mt.match_features(described(arr_a), described(arr_b), R.MatcherConfig(m["delta_s"], m["strategy"]))
            assert np.array_equal([p.ref1 for p in pairs], g[f"{m['tag']}__ref1"]), m["tag"]
            assert np.array_equal([p.ref2 for p in pairs], g[f"{m['tag']}__ref2"]), m["tag"]
            assert np.array_equal(np.array([p.delta for p in pairs]), g[f"{m['tag']}__delta"]), m["tag"]


def test_matcher_c1_scale_against_oracle():
    a, b = scenes.config1_pair(0)
    cfg = R.DescriptorConfig(0.0625, 4, 64, True)
    descs = []
    for im in (a, b):
        t = torch.from_numpy(im).cuda()
        kp = device.detect(t, (16, 32, 64), meta=False)
        descs.append(device.describe(t, kp, cfg)[0])
    r1, r2, dl = device.match(descs[0], descs[1])
    A, B = descs[0].double().cpu().numpy(), descs[1].double().cpu().numpy()
    w1, w2, wd = O.match(A, B)
    assert np.array_equal(r1.cpu().numpy(), w1) and np.array_equal(r2.cpu().numpy(), w2)
    assert np.array_equal(dl.cpu().numpy(), wd)
    assert len(w1) > 500


def test_matcher_f64_random_and_threshold_all():
    rng = np.random.default_rng(3)
    base = rng.random((30, 128))
    base /= np.linalg.norm(base, axis=1, keepdims=True)
    noisy = base + rng.normal(0, 0.01, base.shape)
    pairs = Mt.match_features(described(base), described(noisy), R.MatcherConfig(0.35))
    assert len(pairs) == 30 and all(p.ref1 == p.ref2 for p in pairs)
    w1, w2, wd = O.match(base, noisy)
    assert np.array_equal([p.delta for p in pairs], wd)
    d = np.zeros((2, 128))
    d[0, 0] = 1
    d[1, 0], d[1, 1] = 0.999, 0.01
    tp = Mt.match_features(described(d), described(d), R.MatcherConfig(0.5, "threshold_all"))
    assert {(p.ref1, p.ref2) for p in tp} == {(0, 0), (0, 1), (1, 0), (1, 1)}
    assert Mt.match_features(described(np.zeros((0, 128))), described(d), R.MatcherConfig()) == []


# ---------------------------------------------------------------------------
# P4 -- RANSAC
# ---------------------------------------------------------------------------

def corner_error(m1, m2, nr=768, nc=1024):
    err = 0.0
    for x, y in ((0, 0), (nc - 1, 0), (0, nr - 1), (nc - 1, nr - 1)):
        p = [math.cos(m[0]) * x - math.sin(m[0]) * y + m[1] for m in (m1, m2)]
        q = [math.sin(m[0]) * x + math.cos(m[0]) * y + m[2] for m in (m1, m2)]
        err = max(err, math.hypot(p[0] - p[1], q[0] - q[1]))
    return err


def test_ransac_matches_reference_fixtures(golden):
    g = golden("ransac.npz")
    meta = json.loads(str(g["meta"]))
    for m in meta["cases"]:
        lab = m["label"]
        src, dst = g[f"{lab}__src"], g[f"{lab}__dst"]
        cfg = R.RansacConfig(m["iterations"], m["inlier_tol"], m["min_inliers"], m["seed"])
        if not bool(g[f"{lab}__ok"]):
            with pytest.raises(RegistrationError):
                Rg.ransac_points(src, dst, cfg)
            continue
        res = Rg.ransac_points(src, dst, cfg)
        assert res.inliers == g[f"{lab}__inliers"].tolist(), lab
        assert res.consensus_size == int(g[f"{lab}__consensus"]), lab
        want = g[f"{lab}__model"]
        assert corner_error((res.transform.theta, res.transform.t_x, res.transform.t_y), want) <= 1e-3, lab
    for k in meta["est"]:
        t = Rg.estimate_rigid(g[f"est{k}__src"], g[f"est{k}__dst"])
        assert corner_error((t.theta, t.t_x, t.t_y), g[f"est{k}__model"]) <= 1e-6


def test_estimate_rigid_kats():
    t = Rg.estimate_rigid([(1, 0), (0, 1)], [(5, -2), (4, -3)])
    assert t.theta == pytest.approx(math.pi / 2, abs=1e-12)
    assert (t.t_x, t.t_y) == pytest.approx((5, -3), abs=1e-12)
    t0 = Rg.estimate_rigid([(0, 0), (1, 0)], [(0, 0), (1, 0)])
    assert t0.theta == 0.0 and (t0.t_x, t0.t_y) == (0.0, 0.0)
    with pytest.raises(DegenerateSampleError):
        Rg.estimate_rigid([(1, 1)], [(2, 2)])
    with pytest.raises(DegenerateSampleError):
        Rg.estimate_rigid([(1, 1), (1, 1)], [(0, 0), (5, 5)])


# ---------------------------------------------------------------------------
# P5 -- end to end (small pair through the reference chain)
# ---------------------------------------------------------------------------

def test_end_to_end_small_pair(golden):
    from paper_2405_08578_b200.pipeline import PipelineConfig, prepare_image, register_prepared

    g = golden("e2e.npz")
    cfg = PipelineConfig(window_min=16, window_max=64, ransac_iters=1000)
    preps = []
    for tag in ("a", "b"):
        p = prepare_image(R.IntensityImage(g[tag], tag), cfg)
        h = p.keypoints.image(0)
        h["pol"] = h.pop("polarity")
        assert_kp_equal(h, {f: g[f"{tag}__{f}"] for f in KP}, tag)
        ref = g[f"{tag}__desc"]
        got = p.descriptors.double().cpu().numpy()
        rel = np.max(np.abs(got - ref), axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-300)
        assert rel.max() <= P2_TOL
        preps.append(p)
    pairs, res, _, _ = register_prepared(preps[0], preps[1], cfg)
    assert res is not None
    # P5: every match-set difference is a near-tie of the reference's distance
    # matrix under the measured descriptor perturbation (tests/match_diff.py)
    want_pairs = set(zip(g["m__ref1"].tolist(), g["m__ref2"].tolist()))
    got_pairs = {(p.ref1, p.ref2) for p in pairs}
    Ar, Br = (g[f"{t}__desc"].astype(np.float32).astype(np.float64) for t in "ab")  # the golden matched fp32 rows
    (w1, w2, _), stats = ref_match_with_gaps(Ar, Br, cfg.delta_s)
    assert set(zip(w1.tolist(), w2.tolist())) == want_pairs  # the classifier's matrix is the reference's
    cls = classify(Ar, Br, *(p.descriptors.double().cpu().numpy() for p in preps), want_pairs, got_pairs,
                   cfg.delta_s, stats)
    assert cls["others"] == [], cls
    assert len(want_pairs ^ got_pairs) <= 0.02 * len(want_pairs)
    assert corner_error((res.transform.theta, res.transform.t_x, res.transform.t_y), g["r__model"], 384, 400) <= 1e-3


# ---------------------------------------------------------------------------
# P3 on the tensor-core path (forced on for small problems)
# ---------------------------------------------------------------------------

def test_matcher_tc_path_matches_reference_fixtures(golden):
    g = golden("matcher.npz")
    for m in json.loads(str(g["meta"])):
        if m["strategy"] != "nearest_neighbor":
            continue
        A, B = g[f"{m['label']}__A"], g[f"{m['label']}__B"]
        if len(A) == 0 or len(B) == 0:
            continue
        for arr_a, arr_b in ((A, B), (A.astype(np.float64), B.astype(np.float64))):
            r1, r2, dl = device.match(torch.from_numpy(arr_a).cuda(), torch.from_numpy(arr_b).cuda(), m["delta_s"],
                                      path="tensor")
            assert np.array_equal(r1.cpu().numpy(), g[f"{m['tag']}__ref1"]), m["tag"]
            assert np.array_equal(r2.cpu().numpy(), g[f"{m['tag']}__ref2"]), m["tag"]
            assert np.array_equal(dl.cpu().numpy(), g[f"{m['tag']}__delta"]), m["tag"]


def test_matcher_tc_near_duplicate_clusters():
    """Clusters of bit-identical and of 1-ulp-apart rows: top-4 overflow, the
    tensor-core enumeration of near-ties and the exact decision all engage."""
    rng = np.random.default_rng(11)
    base = rng.random((40, 128)).astype(np.float32)
    base /= np.linalg.norm(base, axis=1, keepdims=True)
    rows_a, rows_b = [], []
    for c in range(40):
        for _ in range(int(rng.integers(1, 30))):
            v = base[c].copy()
            if rng.random() < 0.5:  # perturb a few elements by one ulp
                k = rng.integers(0, 128, size=3)
                v[k] = np.nextafter(v[k], np.float32(2.0))
            rows_a.append(v)
        for _ in range(int(rng.integers(1, 30))):
            v = base[c] + (rng.normal(0, 0.02, 128).astype(np.float32) if rng.random() < 0.3 else 0)
            rows_b.append(v.astype(np.float32))
    A, B = np.stack(rows_a), np.stack(rows_b)
    A, B = A[rng.permutation(len(A))], B[rng.permutation(len(B))]
    r1, r2, dl = device.match(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), path="tensor")
    w1, w2, wd = O.match(A.astype(np.float64), B.astype(np.float64))
    assert np.array_equal(r1.cpu().numpy(), w1) and np.array_equal(r2.cpu().numpy(), w2)
    assert np.array_equal(dl.cpu().numpy(), wd)
    assert len(w1) >= 20


def test_float_grey_raster_path_matches_oracle():
    """BT.601 grey (non-integral float64) rasters: detection on the recomputed
    float64 P with first-occurrence ties, descriptors by the float64 kernel."""
    rgb = np.stack([scenes.scene(200, 320, 50 + c) for c in range(3)], axis=-1)
    grey = scenes.gray_bt601(rgb)
    alpha = O.default_alpha(*grey.shape)
    P = O.ramp(grey, alpha)
    want = O.detect(P, (16, 32, 64))
    t = torch.from_numpy(grey).cuda()
    kp = device.detect(t, (16, 32, 64), alpha=alpha)
    h = kp.image(0)
    h["pol"] = h.pop("polarity")
    assert_kp_equal(h, want, "grey")
    d = device.describe(t, kp, R.DescriptorConfig(0.0625, 4, 64, True), alpha=alpha, out64=True, out32=False)
    for k in range(0, len(want), 37):
        ref = O.describe_one(P, int(want["row"][k]), int(want["col"][k]), int(want["scale"][k]), 0.0625, 4, 64)
        got = d[0, k].cpu().numpy()
        assert np.max(np.abs(got - ref)) <= P2_TOL * max(np.linalg.norm(ref), 1e-300)


def test_rowshard_single_rank_equals_match_on_c1():
    from paper_2405_08578_b200.rowshard import match_rows_sharded

    a, b = scenes.config1_pair(0)
    cfg = R.DescriptorConfig(0.0625, 4, 64, True)
    ds = []
    for im in (a, b):
        t = torch.from_numpy(im).cuda()
        kp = device.detect(t, (16, 32, 64), meta=False)
        ds.append(device.describe(t, kp, cfg)[0])
    r1, r2, dl = device.match(ds[0], ds[1])
    # two "ranks" emulated sequentially is not possible without a group; world 1 exercises the path
    s1, s2, sd = match_rows_sharded(ds[0], 0, ds[1], 0.35)
    assert torch.equal(s1.cpu(), r1.long().cpu()) and torch.equal(s2.cpu(), r2.long().cpu())
    assert torch.equal(sd.cpu(), dl.cpu())


def test_nearest_matches_oracle_both_paths():
    rng = np.random.default_rng(8)
    X = rng.random((300, 128)).astype(np.float32)
    Y = rng.random((500, 128)).astype(np.float32)
    Y[7] = Y[9]
    for path in ("tensor", "exact"):
        idx, d = device.nearest(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), path=path)
        for i0, D in O.distances(X.astype(np.float64), Y.astype(np.float64)):
            j = np.argmin(D, axis=1)
            assert np.array_equal(idx[i0:i0 + D.shape[0]].cpu().numpy(), j)
            assert np.array_equal(d[i0:i0 + D.shape[0]].cpu().numpy(), D[np.arange(D.shape[0]), j])


@pytest.mark.parametrize("scale", [1e-3, 3.0, 50.0])
def test_nearest_tc_unnormalised_magnitudes(scale):
    """Tensor-core path on unnormalised rows: tiny values (fp16 subnormals in the
    |y|^2 split), moderate ones, and |y|^2 beyond the fp16 range (no
    certificate: every row must fall back to the exact scan)."""
    rng = np.random.default_rng(int(scale * 1000))
    X = (rng.random((260, 128)) * scale).astype(np.float32)
    Y = (rng.random((300, 128)) * scale).astype(np.float32)
    Y[:100] = X[:100] + np.float32(0.01 * scale) * rng.standard_normal((100, 128)).astype(np.float32)
    idx, d = device.nearest(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), path="tensor")
    for i0, D in O.distances(X.astype(np.float64), Y.astype(np.float64)):
        j = np.argmin(D, axis=1)
        assert np.array_equal(idx[i0:i0 + D.shape[0]].cpu().numpy(), j)
        assert np.array_equal(d[i0:i0 + D.shape[0]].cpu().numpy(), D[np.arange(D.shape[0]), j])


def test_end_to_end_c1_against_oracle_chain():
    """P5 at C1 size: keypoints exact, descriptors <= 1e-4, every match-set
    difference classified as a near-tie ("others" = 0, tests/match_diff.py),
    identical RANSAC transform."""
    a, b = scenes.config1_pair(0)
    cfg = R.DescriptorConfig(0.0625, 4, 64, True)
    ref, gpu = [], []
    for im in (a, b):
        P = O.ramp(im.astype(np.float64), O.default_alpha(*im.shape))
        kp = O.detect(P, (16, 32, 64))
        ref.append((kp, O.describe(P, kp, 0.0625, 4, 64, True)))
        t = torch.from_numpy(im).cuda()
        k = device.detect(t, (16, 32, 64), meta=False)
        gpu.append((k, device.describe(t, k, cfg)[0]))
        h = k.image(0)
        assert np.array_equal(h["row"], kp["row"]) and np.array_equal(h["col"], kp["col"])
        g = gpu[-1][1].double().cpu().numpy()
        rel = np.max(np.abs(g - ref[-1][1]), axis=1) / np.maximum(np.linalg.norm(ref[-1][1], axis=1), 1e-300)
        assert rel.max() <= P2_TOL
    Ar, Br = (r[1].astype(np.float32).astype(np.float64) for r in ref)
    (w1, w2, _), stats = ref_match_with_gaps(Ar, Br, 0.35)
    r1, r2, _ = device.match(gpu[0][1], gpu[1][1])
    want, got = set(zip(w1.tolist(), w2.tolist())), set(zip(r1.cpu().numpy().tolist(), r2.cpu().numpy().tolist()))
    # P5: classify every difference; none may be unexplained
    cls = classify(Ar, Br, *(gg[1].double().cpu().numpy() for gg in gpu), want, got, 0.35, stats)
    print(f"P5 C1: {len(want)} reference matches, {cls['diff']} differ: row ties {cls['row_tie']}, "
          f"column ties {cls['col_tie']}, threshold {cls['threshold']}, others {len(cls['others'])}")
    assert cls["others"] == [], cls["others"][:5]
    assert len(got ^ want) <= 0.05 * len(want)
    ref_r = O.ransac(*O.pair_points(w1, w2, ref[0][0], ref[1][0]), 1000, 3.0, 8, 0)
    src, dst = device.pair_points(r1, r2, gpu[0][0].row[0], gpu[0][0].col[0], gpu[1][0].row[0], gpu[1][0].col[0])
    out = device.ransac(src, dst, 1000, 3.0, 8, 0)
    assert out.ok
    assert corner_error((out.theta, out.t_x, out.t_y), ref_r["model"]) <= 1e-3


# ---------------------------------------------------------------------------
# §8(f) #2: compositor on the device, bit-exact against the reference
# ---------------------------------------------------------------------------

def test_compositor_matches_reference_fixtures(golden):
    from paper_2405_08578_b200 import compositor as K

    g = golden("compositor.npz")
    n = 0
    for m in json.loads(str(g["meta"])):
        ids = [f"i{k}" for k in range(len(m["transforms"]))]
        imgs = {i: g[f"{m['label']}__img{k}"] for k, i in enumerate(ids)}
        pl = [K.Placement(i, R.RigidTransform(*t)) for i, t in zip(ids, m["transforms"])]
        canvas = K.compute_canvas(pl, {i: a.shape for i, a in imgs.items()})
        out = K.warp_and_blend(imgs, pl, canvas, blend=m["blend"], resample=m["resample"])
        assert np.array_equal(out, g[f"{m['label']}__pixels"]), m["label"]
        assert np.array_equal(canvas.weightmap, g[f"{m['label']}__weightmap"]), m["label"]
        n += 1
    assert n >= 10


def test_compositor_reference_properties():
    """The reference's compositor tests (test_compositor.py) on the device path."""
    from paper_2405_08578_b200 import compositor as K

    I = R.RigidTransform.identity()
    rng = np.random.default_rng(0)
    px = rng.uniform(0, 255, size=(40, 60))
    c = K.compute_canvas([K.Placement("a", I)], {"a": px.shape})
    assert np.array_equal(K.warp_and_blend({"a": px}, [K.Placement("a", I)], c), px)  # identity bit-exact
    c = K.compute_canvas([K.Placement("a", I)], {"a": px.shape})
    assert np.array_equal(K.warp_and_blend({"a": px}, [K.Placement("a", I)], c, resample="nearest"), px)
    pl = [K.Placement("a", I), K.Placement("b", R.RigidTransform(0.0, 80.0, 0.0))]
    flat = np.full((40, 40), 200.0)
    c = K.compute_canvas(pl, {"a": (40, 40), "b": (40, 40)})
    out = K.warp_and_blend({"a": flat, "b": flat}, pl, c)
    assert (c.height, c.width) == (40, 120)
    assert np.all(out[:, 41:79] == 0.0) and np.all(c.weightmap[:, 41:79] == 0.0)
    assert np.all(c.weightmap[:, :40] > 0.0)
    a, b = np.full((20, 20), 10.0), np.full((20, 20), 250.0)
    pl = [K.Placement("a", I), K.Placement("b", I)]
    c = K.compute_canvas(pl, {"a": a.shape, "b": b.shape})
    assert np.all(K.warp_and_blend({"a": a, "b": b}, pl, c, blend="overwrite") == 250.0)
    with pytest.raises(ValueError):
        K.warp_and_blend({"a": a}, [K.Placement("a", I)], c, blend="average")
    with pytest.raises(ValueError):
        K.warp_and_blend({"a": a}, [K.Placement("a", I)], c, resample="cubic")


def test_compositor_many_placements_carry_state_between_launches():
    """More placements than one kernel-parameter batch (64): the per-pixel
    state crosses launches; result still equals the oracle bit for bit."""
    from paper_2405_08578_b200 import compositor as K

    rng = np.random.default_rng(3)
    imgs, tr = [], []
    for k in range(70):
        imgs.append(rng.uniform(0, 255, size=(12, 16)))
        tr.append((float(rng.uniform(-0.3, 0.3)), float(rng.uniform(0, 40)), float(rng.uniform(0, 30))))
    ids = [f"i{k}" for k in range(70)]
    pl = [K.Placement(i, R.RigidTransform(*t)) for i, t in zip(ids, tr)]
    canvas = K.compute_canvas(pl, {i: a.shape for i, a in zip(ids, imgs)})
    out = K.warp_and_blend(dict(zip(ids, imgs)), pl, canvas)
    bounds = O.canvas_bounds(tr, [a.shape for a in imgs])
    want, wm = O.composite(imgs, tr, bounds)
    assert np.array_equal(out, want) and np.array_equal(canvas.weightmap, wm)


# ---------------------------------------------------------------------------
# §8(f) #3: RGB ingest on the device (integer luma key, host grey table)
# ---------------------------------------------------------------------------

def test_rgb_ingest_grey_detect_describe_match_oracle():
    """C5-size RGB image: device grey == reference to_grayscale bits;
    keypoints (integer luma key) bit-exact against the oracle on that grey;
    descriptors identical to the float64-grey path's and <= 1e-4 from the oracle."""
    from paper_2405_08578_b200 import ingest

    a, b, _ = scenes.config5_pair(1)
    grey = scenes.gray_bt601(a)
    ta = torch.from_numpy(a).cuda()
    assert np.array_equal(ingest.to_grayscale_device(ta).cpu().numpy(), grey)
    alpha = O.default_alpha(*grey.shape)
    want = O.detect(O.ramp(grey, alpha), (16, 32, 64))
    im_rgb = device.as_device_images(ta, alpha, rgb=True)
    kp = device.detect(im_rgb, (16, 32, 64))
    h = kp.image(0)
    h["pol"] = h.pop("polarity")
    assert_kp_equal(h, want, "rgb")
    cfg = R.DescriptorConfig(0.0625, 4, 64, True)
    d_rgb = device.describe(im_rgb, kp, cfg, out64=True, out32=False)
    tg = torch.from_numpy(grey).cuda()
    kp_g = device.detect(tg, (16, 32, 64), alpha=alpha)
    assert torch.equal(kp_g.row, kp.row) and torch.equal(kp_g.value, kp.value)
    d_g = device.describe(tg, kp_g, cfg, alpha=alpha, out64=True, out32=False)
    # same raster bits; the RGB8 fast kernel's 52-bit histograms vs the general kernel's 63-bit
    rel = (d_rgb - d_g).abs().amax(dim=-1) / d_g.norm(dim=-1).clamp_min(1e-300)
    assert float(rel.max()) <= 1e-12
    P = O.ramp(grey, alpha)
    for k in range(0, len(want), 211):
        ref = O.describe_one(P, int(want["row"][k]), int(want["col"][k]), int(want["scale"][k]), 0.0625, 4, 64)
        got = d_rgb[0, k].cpu().numpy()
        assert np.max(np.abs(got - ref)) <= P2_TOL * max(np.linalg.norm(ref), 1e-300)


def test_rgb_batch_and_tiny_alpha_float_compare():
    """RGB batches use per-image offsets of 3 bytes per pixel; an alpha below
    the key rule falls back to the exact float64 compare on the table grey."""
    rng = np.random.default_rng(21)
    imgs = rng.integers(0, 256, size=(3, 96, 120, 3)).astype(np.uint8)
    imgs[1, 10:40, 20:70] = (12, 200, 77)  # flat region: ties resolved by the ramp
    for alpha in (O.default_alpha(96, 120), 1e-14):
        kp = device.detect(torch.from_numpy(imgs).cuda(), (8, 16), alpha=alpha)
        for i in range(3):
            want = O.detect(O.ramp(scenes.gray_bt601(imgs[i]), alpha), (8, 16))
            h = kp.image(i)
            h["pol"] = h.pop("polarity")
            assert_kp_equal(h, want, f"rgb{i}/{alpha}")


def test_rgb_table_and_formula_modes_agree():
    """The RGB8 kernels read the grey from the host-built table or -- when
    ps_gray_table_check finds the two-FMA formula equal to it on all 2^24
    triples -- compute it; both give identical keypoints and descriptors."""
    from paper_2405_08578_b200 import ingest

    a, _, _ = scenes.config5_pair(2)
    t = torch.from_numpy(a).cuda().unsqueeze(0)
    alpha = O.default_alpha(a.shape[0], a.shape[1])
    auto = device.as_device_images(t, alpha, rgb=True)
    table = device.DeviceImages(t, "rgb8", alpha, ingest.gray_lut(t.device))
    cfg = R.DescriptorConfig(0.0625, 4, 64, True)
    k1, k2 = device.detect(auto, (16, 32, 64)), device.detect(table, (16, 32, 64))
    assert torch.equal(k1.row, k2.row) and torch.equal(k1.col, k2.col) and torch.equal(k1.value, k2.value)
    d1 = device.describe(auto, k1, cfg, out64=True, out32=False)
    d2 = device.describe(table, k2, cfg, out64=True, out32=False)
    assert torch.equal(d1, d2)
    g = ingest.to_grayscale_device(t)[0].cpu().numpy()
    assert np.array_equal(g, scenes.gray_bt601(a))


def test_describe_pair_and_single_kernels_agree():
    """The two-keypoints-per-warp kernel and the one-keypoint kernel compute
    the same descriptors (to float64 rounding) -- on a full C2 image (even
    counts) and on a deduplicated multi-scale list with an odd count (a
    half-idle last warp)."""
    img = scenes.scene(640, 960, 3)
    t = torch.from_numpy(img).cuda()
    cfg = R.DescriptorConfig(0.0625, 4, 64, True)
    for scales, meta in (((8, 16, 32), False), ((8, 12, 24), True)):
        kp = device.detect(t, scales, meta=meta)
        if meta and int(kp.count[0]) % 2 == 0:
            kp.count[0] -= 1  # an odd count: the last warp has one live half
        d_pair = device.describe(t, kp, cfg, scale_set=kp.scale_set, out64=True, out32=False)
        d_one = device.describe(t, kp, cfg, scale_set=kp.scale_set, out64=True, out32=False, policy="single")
        n = int(kp.count[0])
        a, b = d_pair[0, :n], d_one[0, :n]
        rel = (a - b).abs().amax(dim=-1) / b.norm(dim=-1).clamp_min(1e-300)
        assert float(rel.max()) <= 1e-12, (scales, float(rel.max()))
        assert torch.all((a.norm(dim=-1) - 1).abs() < 1e-9)


def test_host_batch_pipeline_grey_and_rgb():
    """pipeline.prepare_batch_host (pinned host in/out, 3-stream pipeline) gives
    the device path's keypoints and descriptors, for grey and RGB batches
    (5 images, chunk 2: partial last chunk, slot reuse)."""
    from paper_2405_08578_b200 import pipeline as PL

    cfg = PL.PipelineConfig(window_min=16, window_max=64)
    grey = np.stack([scenes.scene(200, 288, s) for s in range(5)])
    rgb = np.stack([np.stack([scenes.scene(200, 288, 10 * s + c) for c in range(3)], axis=-1) for s in range(5)])
    for imgs in (grey, rgb):
        out = PL.prepare_batch_host(torch.from_numpy(imgs).pin_memory(), cfg, chunk=2)
        dimg = device.as_device_images(torch.from_numpy(imgs).cuda(), rgb=imgs.ndim == 4)
        kp = device.detect(dimg, cfg.scale_set().sizes, meta=False)
        d = device.describe(dimg, kp, cfg.descriptor_config(), scale_set=kp.scale_set)
        for b in range(5):
            n = int(out.count[b])
            assert n == int(kp.count[b])
            assert np.array_equal(out.row[b, :n].numpy(), kp.row[b, :n].cpu().numpy())
            assert np.array_equal(out.value[b, :n].numpy(), kp.value[b, :n].cpu().numpy())
            assert np.array_equal(out.descriptors[b, :n].numpy(), d[b, :n].cpu().numpy())


@pytest.mark.parametrize("n", [2, 3, 8, 97, 1000, 65537, 3 * 2**29 + 5, 2**31 - 1])
def test_sample_stream_on_device_matches_numpy(n):
    """ps_ransac_samples reproduces numpy's PCG64 bounded draws exactly --
    the jump-ahead fast path and the sequential replay (n = 2: one-value
    ranges consume nothing; n near 2^31: frequent Lemire rejections)."""
    for seed in (0, 1, 99, 2**40 + 7):
        for iters in (1, 7, 2000):
            want = device.sample_stream(seed, n, iters)
            got = device.sample_stream_device(seed, n, iters).cpu().numpy()
            assert np.array_equal(got, want), (n, seed, iters)


@pytest.mark.parametrize("scales,l_max", [((32, 64, 128), 128), ((16, 32, 64), 64), ((8, 16, 32), 32)])
def test_fast_describe_kernels_agree_with_general_kernel(scales, l_max):
    """w = 8 (pair kernel) and w = 16 (the reference's default 32..128
    windows) fast kernels against the general float64 kernel, and a sample
    against the oracle."""
    img = scenes.scene(700, 900, 21)
    t = torch.from_numpy(img).cuda()
    cfg = R.DescriptorConfig(0.0625, 4, l_max, True)
    kp = device.detect(t, scales, meta=False)
    d_fast = device.describe(t, kp, cfg, scale_set=kp.scale_set, out64=True, out32=False)
    d_gen = device.describe(t, kp, cfg, scale_set=kp.scale_set, out64=True, out32=False, policy="general")
    n = int(kp.count[0])
    a, b = d_fast[0, :n], d_gen[0, :n]
    rel = (a - b).abs().amax(dim=-1) / b.norm(dim=-1).clamp_min(1e-300)
    # the general kernel screens 8-bit rasters with float32 magnitudes (~1e-7)
    assert float(rel.max()) <= 1e-6, float(rel.max())
    alpha = O.default_alpha(*img.shape)
    P = O.ramp(img.astype(np.float64), alpha)
    h = kp.image(0)
    for k in range(0, n, max(1, n // 40)):
        ref = O.describe_one(P, int(h["row"][k]), int(h["col"][k]), scales[0], 0.0625, 4, l_max)
        assert np.max(np.abs(a[k].cpu().numpy() - ref)) <= P2_TOL * max(np.linalg.norm(ref), 1e-300)


def test_stitch_pair_and_plan_and_stitch_on_device():
    """pipeline.stitch_pair and mosaic.plan_and_stitch (the callers of the
    path, with the device compositor): crops of one scene register at their
    true offsets and the composite reproduces the scene where it is covered."""
    from paper_2405_08578_b200 import mosaic, pipeline as PL

    src = scenes.scene(360, 480, 11).astype(np.float64)
    cfg = PL.PipelineConfig(window_min=16, window_max=64, seed=7)
    a = R.IntensityImage(src[:, :300].copy(), "a")
    b = R.IntensityImage(src[:, 180:].copy(), "b")
    res = PL.stitch_pair(a, b, cfg)
    assert res.success and res.report["matched_pairs"] > 50
    # the transform maps a's pixels onto b: x_b = x_a - 180
    assert abs(res.transform.t_x + 180) < 0.5 and abs(res.transform.t_y) < 0.5
    assert res.composite.shape == (360, 480)
    cov = res.composite != 0  # a ~1e-19 rad rotation can leave a border column uncovered (as in the reference)
    assert cov.mean() > 0.99
    assert float(np.sqrt(np.mean((res.composite[cov] - src[cov]) ** 2))) < 1.0
    frags, offs = [], {}
    for k, (r0, c0) in enumerate([(0, 0), (0, 200), (140, 0), (140, 200)]):
        frags.append(R.IntensityImage(src[r0:r0 + 220, c0:c0 + 280].copy(), f"f{k}"))
        offs[f"f{k}"] = (r0, c0)
    plan, comp = mosaic.plan_and_stitch(frags, cfg)
    assert plan.final_unmatched == []
    ref = plan.rounds[0].reference_id
    assert comp.shape == (360, 480)
    cov = comp != 0
    assert cov.mean() > 0.99
    assert float(np.sqrt(np.mean((comp[cov] - src[cov]) ** 2))) < 1.0, ref


def test_match_many_and_ransac_many_equal_single_calls(monkeypatch):
    """The batched, synchronisation-free pair path (ps_match_async through
    device.match_many, device.ransac_many) gives exactly the results of the
    one-pair calls and of the oracle, on one stream and spread over streams:
    tensor-core pairs of C1 crops, a near-duplicate cluster pair (top-4
    overflow + enumeration), an empty side, a CUDA-core (small) pair."""
    cfg = R.DescriptorConfig(0.0625, 4, 64, True)
    descs, kps = [], []
    for p in range(2):
        a, b = scenes.config1_pair(p)
        for im in (a, b):
            t = torch.from_numpy(im).cuda()
            kp = device.detect(t, (16, 32, 64), meta=False)
            kps.append(kp)
            descs.append(device.describe(t, kp, cfg)[0])
    rng = np.random.default_rng(5)
    base = rng.random((12, 128)).astype(np.float32)
    A = np.repeat(base, 20, axis=0)
    A[::3, 5] = np.nextafter(A[::3, 5], np.float32(2))
    B = base[rng.integers(0, 12, 200)] + np.where(rng.random((200, 1)) < 0.3, 0.01, 0).astype(np.float32)
    small = torch.from_numpy(rng.random((40, 128)).astype(np.float32)).cuda()
    # > 512 distinct rows with near-tied candidates: beyond the blind
    # enumeration row blocks of the asynchronous mode, the exact scan decides
    cl = base[rng.integers(0, 12, 1500)].copy()
    cl[np.arange(1500), rng.integers(0, 128, 1500)] += np.float32(1e-6)
    cb = base[rng.integers(0, 12, 900)].copy()
    cb[np.arange(900), rng.integers(0, 128, 900)] -= np.float32(1e-6)
    pairs = [(descs[0], descs[1]), (descs[2], descs[3]), (descs[0], descs[3]),
             (torch.from_numpy(A).cuda(), torch.from_numpy(B.astype(np.float32)).cuda()),
             (descs[0][:0], descs[1]), (small, small.flip(0)),
             (torch.from_numpy(cl).cuda(), torch.from_numpy(cb).cuda())]
    for streams in (None, [torch.cuda.Stream() for _ in range(3)]):
        got = device.match_many(pairs, 0.35, streams=streams)
        for q, ((x, y), (r1, r2, dl)) in enumerate(zip(pairs, got)):
            s1, s2, sd = device.match(x, y)
            assert torch.equal(r1, s1) and torch.equal(r2, s2) and torch.equal(dl, sd), q
            if q in (0, 3, 5, 6):
                w1, w2, wd = O.match(x.double().cpu().numpy(), y.double().cpu().numpy())
                assert np.array_equal(r1.cpu().numpy(), w1) and np.array_equal(dl.cpu().numpy(), wd), q
    # RANSAC of the registered C1 pairs, batched vs one call each
    got = device.match_many(pairs[:2], 0.35)
    jobs = []
    for q, (r1, r2, _) in enumerate(got):
        k1, k2 = kps[2 * q], kps[2 * q + 1]
        src, dst = device.pair_points(r1, r2, k1.row[0], k1.col[0], k2.row[0], k2.col[0])
        jobs.append((src, dst, 1000, 3.0, 8, 10 + q))
    for streams in (None, [torch.cuda.Stream() for _ in range(2)]):
        many = device.ransac_many(jobs, streams=streams)
        for (src, dst, it, tol, mi, seed), o in zip(jobs, many):
            one = device.ransac(src, dst, it, tol, mi, seed)
            assert o.ok and one.ok and np.array_equal(o.inliers, one.inliers)
            assert (o.theta, o.t_x, o.t_y, o.rms, o.consensus) == (one.theta, one.t_x, one.t_y, one.rms, one.consensus)
            ref = O.ransac(src.cpu().numpy(), dst.cpu().numpy(), it, tol, mi, seed)
            assert np.array_equal(o.inliers, ref["inliers"])


def test_pairwise_table_batched_equals_per_pair():
    """build_pairwise_table with the batched engine (two host syncs for all
    pairs) and with one pair at a time give the same table."""
    from paper_2405_08578_b200 import mosaic, pipeline as PL

    src = scenes.scene(420, 560, 21)
    cfg = PL.PipelineConfig(window_min=16, window_max=64, seed=3)
    frags = [src[r0:r0 + 260, c0:c0 + 340].copy() for r0, c0 in [(0, 0), (0, 220), (160, 0), (160, 220), (80, 110)]]
    t1 = mosaic.build_pairwise_table(frags, cfg, engine=mosaic.GpuEngine(cfg, batched=True, n_streams=3))
    t2 = mosaic.build_pairwise_table(frags, cfg, engine=mosaic.GpuEngine(cfg, batched=False))
    ge = mosaic.GraphEngine(cfg, n_streams=3)
    t3 = mosaic.build_pairwise_table(frags, cfg, engine=ge)  # eager warm-up + capture
    t4 = mosaic.build_pairwise_table(frags, cfg, engine=ge)  # graph replays
    other = [f[::-1].copy() for f in frags]  # new pixels through the same graphs
    t5 = mosaic.build_pairwise_table(other, cfg, engine=ge)
    t6 = mosaic.build_pairwise_table(other, cfg, engine=mosaic.GpuEngine(cfg, batched=False))
    assert t1.entries.keys() == t2.entries.keys() and len(t1.entries) >= 8
    for ta, tb in ((t1, t2), (t3, t2), (t4, t2), (t5, t6)):
        assert ta.entries.keys() == tb.entries.keys()
        for k, e in ta.entries.items():
            f = tb.entries[k]
            assert e.inlier_count == f.inlier_count
            assert (e.transform.theta, e.transform.t_x, e.transform.t_y) == \
                   (f.transform.theta, f.transform.t_x, f.transform.t_y)


def test_ransac_with_device_count_equals_host_count():
    """ps_ransac_rigid_async reads the correspondence count on the device:
    same result as the host-count call for the prefix of a larger buffer, and
    PS_ERR_REGISTRATION in the status word when the count is below
    min_inliers (registration.py:158-162)."""
    from paper_2405_08578_b200 import _lib

    rng = np.random.default_rng(2)
    n = 900
    src = rng.uniform(0, 800, (n, 2))
    th = 0.1
    R2 = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
    dst = src @ R2.T + [20.0, -7.0] + rng.normal(0, 0.8, (n, 2))
    dst[::3] = rng.uniform(0, 800, (len(dst[::3]), 2))
    S, D = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
    for m, seed in ((900, 0), (437, 5), (9, 1), (5, 2), (1, 3), (0, 4)):
        cnt = torch.tensor([m], dtype=torch.int64, device="cuda")
        out = torch.zeros(8 + (n + 7) // 8, dtype=torch.float64, device="cuda")
        device.ransac_async_dev(S, D, cnt, n, 700, 3.0, 8, seed, out)
        got = device.ransac_result(out.cpu(), m)
        if m < 8:
            assert got.status == _lib.PS_ERR_REGISTRATION and not got.ok, m
            continue
        one = device.ransac(S[:m], D[:m], 700, 3.0, 8, seed)
        assert got.ok == one.ok and np.array_equal(got.inliers, one.inliers), m
        assert (got.theta, got.t_x, got.t_y, got.rms, got.consensus) == (one.theta, one.t_x, one.t_y, one.rms,
                                                                          one.consensus)


def test_graph_engine_device_batch_rgb_pairs_equal_sequential():
    """GraphEngine.prepare_device (RGB batch, replayed graph) + register_many
    (replayed pair graph) give the per-pair sequential results on small C5-style
    pairs, on the capture call and on replays."""
    from paper_2405_08578_b200 import mosaic
    from paper_2405_08578_b200.pipeline import PipelineConfig

    cfg = PipelineConfig(window_min=16, window_max=64, ransac_iters=500)
    pairs = [scenes.config5_pair(p, 270, 480)[:2] for p in range(3)]
    pairs.append((pairs[0][0], pairs[0][0].copy()))  # an identical pair registers exactly
    rgb = torch.from_numpy(np.stack([im for pr in pairs for im in pr])).cuda()
    imgs = device.as_device_images(rgb, rgb=True)
    sizes, dcfg = cfg.scale_set().sizes, cfg.descriptor_config()
    kp = device.detect(imgs, sizes, meta=False)
    d = device.describe(imgs, kp, dcfg, scale_set=kp.scale_set)
    want = []
    for q in range(len(pairs)):
        r1, r2, _ = device.match(d[2 * q], d[2 * q + 1])
        if int(r1.shape[0]) < cfg.min_inliers:
            want.append((False, 0.0, 0.0, 0.0, 0))
            continue
        src, dst = device.pair_points(r1, r2, kp.row[2 * q], kp.col[2 * q], kp.row[2 * q + 1], kp.col[2 * q + 1])
        o = device.ransac(src, dst, cfg.ransac_iters, cfg.ransac_tol, cfg.min_inliers, cfg.seed)
        want.append((True, o.theta, o.t_x, o.t_y, int(o.inliers.shape[0])) if o.ok else (False, 0.0, 0.0, 0.0, 0))
    eng = mosaic.GraphEngine(cfg, n_streams=3)
    for _ in range(3):  # capture, then replays
        rows, cols, desc, cnt = eng.prepare_device(imgs)
        h = cnt.cpu().tolist()
        R, Cc, Dd = rows.unbind(0), cols.unbind(0), desc.unbind(0)
        items = [(R[2 * q], Cc[2 * q], Dd[2 * q], h[2 * q], R[2 * q + 1], Cc[2 * q + 1], Dd[2 * q + 1], h[2 * q + 1],
                  cfg.seed) for q in range(len(pairs))]
        assert eng.register_many(items) == want
    assert want[-1][0] and want[-1][4] > 100  # the identical pair


def test_descriptor_out_of_image_features_clamped_like_reference():
    """The reference translates the region inward for any feature position
    (descriptor.py:118-131, 237-239) -- even outside the image; the drop-in
    does the same (u8 fast kernels queue such keypoints for the general one)."""
    img = scenes.scene(120, 150, 9)
    alpha = O.default_alpha(*img.shape)
    P = O.ramp(img.astype(np.float64), alpha)
    rimg = R.apply_linear_ramp(R.IntensityImage(img, "x"), alpha)
    cfg = R.DescriptorConfig(0.0625, 4, 64, True)
    pts = [(-5, 3), (0, 0), (119, 149), (130, 160), (60, -40), (-1000, 2000), (50, 75)]
    feats = [R.FeaturePoint(r, c, s, "max", 0, 0.0) for r, c in pts for s in (16, 32, 64)]
    got = Dsc.describe_features(rimg, feats, cfg).descriptors
    for k, f in enumerate(feats):
        ref = O.describe_one(P, f.row, f.col, f.scale, 0.0625, 4, 64)
        assert np.max(np.abs(got[k] - ref)) <= P2_TOL * max(np.linalg.norm(ref), 1e-300), f


@pytest.mark.parametrize("nr,nc,scales", [(97, 131, (16, 24)), (200, 333, (36,)), (150, 255, (8, 12, 40)),
                                          (64, 64, (17,)), (300, 257, (32, 64, 128)), (130, 140, (8, 16, 32)),
                                          (250, 300, (48,)), (300, 1200, (48, 80)), (150, 2000, (36,)),
                                          (100, 1700, (20,)), (330, 900, (96, 100)), (400, 700, (160, 176)),
                                          (75, 5000, (36, 37))])
def test_strip_detector_padded_pitch_tie_heavy(nr, nc, scales):
    """The vectorised strip kernel (any window side, 16-byte aligned rows):
    tie-heavy u8 and RGB rasters in a padded-pitch layout (odd widths, shrunk
    trailing windows, non-nested and nested scale sets) against the oracle."""
    rng = np.random.default_rng(nr * nc)
    pitch = (nc + 15) // 16 * 16 + 16
    px = (rng.integers(0, 3, size=(2, nr, nc)) * 100).astype(np.uint8)
    buf = torch.zeros((2, nr, pitch), dtype=torch.uint8, device="cuda")
    buf[:, :, :nc] = torch.from_numpy(px).cuda()
    alpha = O.default_alpha(nr, nc)
    kp = device.detect(device.DeviceImages(buf[:, :, :nc], "u8", alpha), scales)
    rgb = rng.integers(0, 2, size=(2, nr, nc, 3)).astype(np.uint8) * np.uint8(120)
    rbuf = torch.zeros((2, nr, pitch, 3), dtype=torch.uint8, device="cuda")
    rbuf[:, :, :nc] = torch.from_numpy(rgb).cuda()
    from paper_2405_08578_b200.ingest import gray_source

    kr = device.detect(device.DeviceImages(rbuf[:, :, :nc], "rgb8", alpha, gray_source(rbuf.device)), scales)
    for b in range(2):
        want = O.detect(O.ramp(px[b].astype(np.float64), alpha), scales)
        h = kp.image(b)
        h["pol"] = h.pop("polarity")
        assert_kp_equal(h, want, f"u8 {b}")
        want = O.detect(O.ramp(scenes.gray_bt601(rgb[b]), alpha), scales)
        h = kr.image(b)
        h["pol"] = h.pop("polarity")
        assert_kp_equal(h, want, f"rgb {b}")
