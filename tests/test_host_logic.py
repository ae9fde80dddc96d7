"""Host-side logic of the package (no GPU): value types, config validation,
region sizes and the RANSAC sample stream, checked against the oracle and
the reference fixtures."""

import json
import math

import numpy as np
import pytest

from oracle import lpsift_oracle as O
from paper_2405_08578_b200 import records as R
from paper_2405_08578_b200.device import sample_stream
from paper_2405_08578_b200.errors import ConfigError
from paper_2405_08578_b200.pipeline import PipelineConfig, pair_seed


def test_scale_set_rules():
    assert R.ScaleSet.from_range(32, 40).sizes == (32, 40)
    assert R.ScaleSet.from_range(8, 64).sizes == (8, 16, 32, 64)
    assert R.ScaleSet.from_range(32, 32).sizes == (32,)
    for bad in [(16, 16), (32, 16), (4,), ()]:
        with pytest.raises(ConfigError):
            R.ScaleSet(bad)
    with pytest.raises(ConfigError):
        R.ScaleSet.from_range(64, 32)
    R.ScaleSet((8, 9, 128))


def test_partition_windows_geometry():
    w = R.partition_windows(70, 64, 32)
    assert [x.height for x in w] == [32, 32, 32, 32, 6, 6]
    assert len(R.partition_windows(50, 83, 16)) == R.window_count(50, 83, 16)


def test_region_size_matches_oracle():
    for beta0, d, lmax in [(0.0625, 4, 128), (0.25, 4, 128), (0.24, 4, 64), (0.0625, 4, 64), (0.1, 3, 40)]:
        cfg = R.DescriptorConfig(beta0, d, lmax)
        for s in range(8, lmax + 1):
            assert R.region_size(s, cfg) == O.region_side(s, beta0, d, lmax)
    assert R.region_size(128, R.DescriptorConfig()) == 32
    assert R.region_size(32, R.DescriptorConfig()) == 16


def test_sample_stream_matches_reference_scalar_calls(golden):
    g = golden("ransac.npz")
    for seed, n in json.loads(str(g["meta"]))["streams"]:
        want = g[f"stream_{seed}_{n}"]
        assert np.array_equal(sample_stream(seed, n, len(want)).astype(np.int64), want)


def test_rigid_transform_algebra():
    t = R.RigidTransform(math.pi / 2, 5, -3)
    assert R.apply_transform(t, (1, 0)) == pytest.approx((5, -2), abs=1e-12)
    assert R.RigidTransform(-math.pi, 0, 0).theta == pytest.approx(math.pi)
    rng = np.random.default_rng(0)
    for _ in range(10):
        a = R.RigidTransform(rng.uniform(-3, 3), rng.uniform(-9, 9), rng.uniform(-9, 9))
        assert np.allclose(a.compose(a.inverse()).matrix, np.eye(3), atol=1e-9)


def test_pipeline_config_validation():
    PipelineConfig(window_min=16, window_max=64)
    PipelineConfig(window_min=8, window_max=128)  # beta0 sits exactly at the bound (C2)
    with pytest.raises(ConfigError):
        PipelineConfig(window_min=4, window_max=16)  # config 4 literal
    with pytest.raises(ConfigError):
        PipelineConfig(beta0=0.5)
    with pytest.raises(ConfigError):
        PipelineConfig(match_strategy="ratio")


def test_pair_seed_is_seedsequence():
    assert pair_seed(0, 1, 2) == int(np.random.SeedSequence([0, 1, 2]).generate_state(1)[0])


def test_apply_linear_ramp_validation_and_lazy_view():
    img = R.IntensityImage(np.full((4, 5), 10.0))
    r = R.apply_linear_ramp(img, 1e-3)
    assert np.array_equal(np.asarray(r.pixels), O.ramp(np.full((4, 5), 10.0), 1e-3))
    with pytest.raises(ConfigError):
        R.apply_linear_ramp(img, 0.0)
    with pytest.raises(ConfigError):
        R.apply_linear_ramp(img, 1.0)


# ---- compositor canvas sizing (host side of §8(f) #2) -------------------------

def test_compute_canvas_matches_reference_cases():
    """The reference's own canvas cases (test_compositor.py) plus the golden
    fixtures' canvases."""
    from paper_2405_08578_b200.compositor import Placement, compute_canvas

    I = R.RigidTransform.identity()
    c = compute_canvas([Placement("a", I)], {"a": (100, 100)})
    assert (c.height, c.width, c.origin_offset) == (100, 100, (0, 0))
    c = compute_canvas([Placement("a", I), Placement("b", R.RigidTransform(0.0, 50.0, 0.0))],
                       {"a": (100, 100), "b": (100, 100)})
    assert (c.height, c.width, c.origin_offset) == (100, 150, (0, 0))
    c = compute_canvas([Placement("a", I), Placement("b", R.RigidTransform(0.0, -30.0, -20.0))],
                       {"a": (100, 100), "b": (100, 100)})
    assert (c.height, c.width, c.origin_offset) == (120, 130, (-30, -20))
    h = 50.0
    quarter = R.RigidTransform(math.pi / 2, h - (math.cos(math.pi / 2) * h - math.sin(math.pi / 2) * h),
                               h - (math.sin(math.pi / 2) * h + math.cos(math.pi / 2) * h))
    c = compute_canvas([Placement("a", I), Placement("b", quarter)], {"a": (100, 100), "b": (100, 100)})
    assert (c.height, c.width) == (100, 100)
    with pytest.raises(ValueError):
        compute_canvas([], {})


def test_compute_canvas_matches_golden(golden):
    from paper_2405_08578_b200.compositor import Placement, compute_canvas

    g = golden("compositor.npz")
    for m in json.loads(str(g["meta"])):
        ids = [f"i{k}" for k in range(len(m["transforms"]))]
        pl = [Placement(i, R.RigidTransform(*t)) for i, t in zip(ids, m["transforms"])]
        dims = {i: g[f"{m['label']}__img{k}"].shape for k, i in enumerate(ids)}
        c = compute_canvas(pl, dims)
        assert [c.width, c.height, *c.origin_offset] == m["canvas"], m["label"]


def test_gray_table_reproduces_reference_to_grayscale():
    """The 2^24-entry grey table (ingest.host_gray_lut) gives the bits of the
    reference's float64 `rgb @ LUMA` (imaging.py:66-68) for whole images of
    awkward sizes (BLAS tails) -- the premise of the RGB8 ingest path."""
    from paper_2405_08578_b200 import ingest, scenes

    lut = ingest.host_gray_lut()
    rng = np.random.default_rng(12)
    for h, w in [(7, 13), (33, 29), (301, 517), (1080, 1920)]:
        img = rng.integers(0, 256, size=(h, w, 3)).astype(np.uint8)
        key = (img[..., 0].astype(np.int64) << 16) | (img[..., 1].astype(np.int64) << 8) | img[..., 2]
        assert np.array_equal(lut[key], scenes.gray_bt601(img)), (h, w)
    a, _, _ = scenes.config5_pair(0)
    key = (a[..., 0].astype(np.int64) << 16) | (a[..., 1].astype(np.int64) << 8) | a[..., 2]
    assert np.array_equal(lut[key], scenes.gray_bt601(a))


# ---- mosaic planning (reference test_mosaic.py table / selection / planning cases) ----

def _chain_table(n):
    from paper_2405_08578_b200.mosaic import PairwiseTransformTable

    table = PairwiseTransformTable(n=n)
    step = R.RigidTransform(0.0, 40.0, 0.0)  # maps (k+1)'s coordinates into k's frame
    for k in range(n - 1):
        table.set_pair(k, k + 1, step, inliers=20)
    return table


def test_mosaic_table_and_reference_selection():
    from paper_2405_08578_b200.mosaic import PairwiseTransformTable, select_reference

    t = _chain_table(3)
    assert t.present(0, 1) and t.present(1, 0) and not t.present(0, 2)
    both = t.get(0, 1).transform.compose(t.get(1, 0).transform)
    assert np.allclose(both.matrix, np.eye(3), atol=1e-6)
    assert select_reference(_chain_table(3), {0, 1, 2}) == 1
    assert select_reference(_chain_table(2), {0, 1}) == 0
    assert select_reference(PairwiseTransformTable(n=6), {5}) == 5
    assert select_reference(_chain_table(4), {1, 2, 3}) == 2


def test_mosaic_planning_cases():
    from paper_2405_08578_b200.mosaic import PairwiseTransformTable, plan_mosaic

    plan, placed = plan_mosaic(_chain_table(2), ["x", "y"])
    assert len(plan.rounds) == 1 and plan.rounds[0].reference_id == "x"
    assert plan.rounds[0].stitched_ids == ["y"] and plan.final_unmatched == []
    assert placed[0] == R.RigidTransform.identity()
    plan, placed = plan_mosaic(_chain_table(4), ["a", "b", "c", "d"])
    assert plan.final_unmatched == [] and set(placed) == {0, 1, 2, 3}
    for k in range(3):
        assert placed[k].t_x - placed[k + 1].t_x == pytest.approx(-40.0, abs=1e-9)
    t = PairwiseTransformTable(n=3)
    t.set_pair(0, 1, R.RigidTransform(0.0, 25.0, 0.0), inliers=15)
    plan, placed = plan_mosaic(t, ["a", "b", "lonely"])
    assert plan.final_unmatched == ["lonely"] and set(placed) == {0, 1}
    t = _chain_table(5)
    t.entries.pop((3, 4))
    t.entries.pop((4, 3))
    plan, _ = plan_mosaic(t, list("abcde"))
    seen = list(plan.final_unmatched)
    for r in plan.rounds:
        seen.append(r.reference_id)
        seen.extend(r.stitched_ids)
    assert sorted(seen) == list("abcde")


def test_plan_and_stitch_argument_errors():
    from paper_2405_08578_b200.mosaic import plan_and_stitch
    from paper_2405_08578_b200.pipeline import PipelineConfig

    cfg = PipelineConfig(window_min=32, window_max=64, seed=7)
    with pytest.raises(ConfigError):
        plan_and_stitch([R.IntensityImage(np.zeros((64, 64)), "solo")], cfg)
    rng = np.random.default_rng(1)
    with pytest.raises(ConfigError):
        plan_and_stitch([R.IntensityImage(rng.uniform(0, 255, (64, 64)), "same"),
                         R.IntensityImage(rng.uniform(0, 255, (64, 64)), "same")], cfg)


def test_axis_sample_36bin_table_is_exact_for_8bit_gradients():
    """csrc/describe_f32.cu g_bin36: for an 8-bit grey raster the axis-sample
    gradient is (da + 2 nc alpha, db + 2 alpha) with integer |da|, |db| <= 255.
    No such integer vector off the axes lies within 1.2e-3 (perpendicular
    distance, gradient units) of a 10-degree bin edge line, so a ramp term
    below 1e-3 cannot move it across one: the reference's bin is the table's.
    On the axes the positive ramp decides (da = 0 < db -> bin 8, db = 0 -> 0)."""
    import math

    import numpy as np

    p, q = np.meshgrid(np.arange(256, dtype=np.float64), np.arange(256, dtype=np.float64), indexing="ij")
    off = (p > 0) & (q > 0)
    edges = np.arange(10) * (2 * math.pi / 36)
    # perpendicular distance of (p, q) to the line at angle e: |q cos e - p sin e|
    dist = np.min(np.abs(q[..., None] * np.cos(edges) - p[..., None] * np.sin(edges)), axis=-1)
    assert dist[off].min() > 1.2e-3
    # table formula vs the reference's float64 arithmetic with a ramp, in all four quadrants
    rng = np.random.default_rng(0)
    tab = np.where((p == 0) & (q > 0), 8, np.floor(np.arctan2(q, p) * (36 / (2 * math.pi)))).astype(int)
    tab[(p == 0) & (q == 0)] = 0
    # (2 nc alpha, 2 alpha): C2, C4, a 13-column image at the 1e-3 limit (flat: atan(1 / nc) < 10 degrees)
    for nc, alpha in [(2688, 5.93e-11), (8192, 3.8e-12), (13, 3.8e-5)]:
        ca, cb = 2 * nc * alpha, 2 * alpha
        da = rng.integers(-255, 256, 20000).astype(np.float64)
        db = rng.integers(-255, 256, 20000).astype(np.float64)
        da[:2000] = 0
        db[2000:4000] = 0
        a, b = da + ca, db + cb
        want = np.minimum((np.mod(np.arctan2(b, a), 2 * math.pi) * (36 / (2 * math.pi))).astype(int), 35)
        t = tab[np.abs(da).astype(int), np.abs(db).astype(int)]
        got = np.where(b < 0, np.where(a < 0, 18 + t, 35 - t), np.where(a < 0, 17 - t, t))
        assert np.array_equal(got, want), (ca, cb)


def test_p5_classifier_explains_perturbation_flips_and_flags_others():
    """tests/match_diff.py (the P5 classifier): its one-pass match equals the
    oracle's, every flip caused by a bounded descriptor perturbation is a
    near-tie, and a pair no tie explains lands in ``others``."""
    from match_diff import classify, ref_match_with_gaps

    rng = np.random.default_rng(5)
    A = rng.random((300, 128))
    A /= np.linalg.norm(A, axis=1, keepdims=True)
    # rows 0..49 have two candidates at nearly equal distance: flips happen
    B = np.concatenate([A[:200] + rng.normal(0, 0.01, (200, 128)), A[:50] + rng.normal(0, 0.01, (50, 128)),
                        rng.random((100, 128))])
    B[250] = B[251]  # an exact column tie
    B /= np.linalg.norm(B, axis=1, keepdims=True)
    (w1, w2, wd), stats = ref_match_with_gaps(A, B, 0.35)
    o1, o2, od = O.match(A, B, 0.35)
    assert np.array_equal(w1, o1) and np.array_equal(w2, o2) and np.array_equal(wd, od)
    Ag = (A + rng.normal(0, 3e-3, A.shape)).astype(np.float32)
    Bg = (B + rng.normal(0, 3e-3, B.shape)).astype(np.float32)
    g1, g2, _ = O.match(Ag.astype(np.float64), Bg.astype(np.float64), 0.35)
    want, got = set(zip(w1.tolist(), w2.tolist())), set(zip(g1.tolist(), g2.tolist()))
    res = classify(A, B, Ag, Bg, want, got, 0.35, stats)
    assert res["diff"] == len(want ^ got) >= 5 and res["others"] == []
    # a far-from-tie pair inserted by hand is not explained
    bad = classify(A, B, A, B, want, got | {(0, 299)}, 0.35, stats)
    assert (0, 299) in {(i, j) for i, j, _ in bad["others"]}
