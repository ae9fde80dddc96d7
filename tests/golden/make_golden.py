"""Generate the golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference (pure Python, numpy) is imported read-only from
``/root/reference/pkg/src``.  Its outputs on seeded inputs are written to
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` pins the oracle to
them and the GPU parity tests compare the CUDA path with them.  Nothing at
test / bench time on the GPU box reads /root/reference.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from peakstitch import descriptor as R_desc  # noqa: E402
from peakstitch import detector as R_det  # noqa: E402
from peakstitch import imaging as R_img  # noqa: E402
from peakstitch import matcher as R_match  # noqa: E402
from peakstitch import registration as R_reg  # noqa: E402
from peakstitch.errors import RegistrationError  # noqa: E402

from paper_2405_08578_b200 import scenes  # noqa: E402

POL = {"max": 0, "min": 1}


def kp_arrays(feats):
    return dict(
        row=np.array([f.row for f in feats], np.int64),
        col=np.array([f.col for f in feats], np.int64),
        scale=np.array([f.scale for f in feats], np.int64),
        pol=np.array([POL[f.polarity] for f in feats], np.int8),
        window=np.array([f.window_index for f in feats], np.int64),
        value=np.array([f.value for f in feats], np.float64),
    )


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)


# --------------------------------------------------------------------------
# detector cases: (label, pixels, alpha, scales, dedupe)
# --------------------------------------------------------------------------

def detector_cases():
    rng = np.random.default_rng(20240514)
    cases = []
    # uint8 tie-heavy content with the pipeline's default alpha
    for k, (nr, nc) in enumerate([(64, 64), (70, 83), (96, 64), (130, 150), (33, 41)]):
        px = rng.integers(0, 4, size=(nr, nc)).astype(np.float64) * 60.0
        for scales in [(8, 16, 32), (8, 9, 33) if min(nr, nc) >= 33 else (8, 9), (16, 32), (32,)]:
            if max(scales) > min(nr, nc):
                continue
            for dd in (True, False):
                cases.append((f"tie{k}_{'_'.join(map(str, scales))}_{int(dd)}", px, None, scales, dd))
    # float uniform (reference tests' style, alpha 1e-5 / 1e-6)
    for k, (nr, nc) in enumerate([(64, 64), (48, 80), (50, 83), (400, 602)]):
        px = rng.uniform(0, 255, size=(nr, nc))
        scales = (16, 32) if nr < 400 else (32, 40)
        cases.append((f"flt{k}", px, 1e-5, scales, True))
    # noise+shapes scene crops, uint8, default alpha; includes (32, 40) and (8,9,128)
    s = scenes.scene(512, 512, 7).astype(np.float64)
    cases.append(("scene_32_40", s[:300, :400], None, (32, 40), True))
    cases.append(("scene_8_9_128", s[:256, :256], None, (8, 9, 128), True))
    cases.append(("scene_16_64_raw", s[:200, :333], None, (16, 32, 64), False))
    cases.append(("constant", np.full((64, 64), 7.0), 1e-5, (32,), True))
    return cases


def make_detector():
    out = {}
    meta = []
    for label, px, alpha, scales, dd in detector_cases():
        nr, nc = px.shape
        a = R_img.default_alpha(nr, nc) if alpha is None else alpha
        rimg = R_img.apply_linear_ramp(R_img.IntensityImage(px, label), a)
        feats = R_det.detect_features(rimg, R_det.ScaleSet(tuple(scales)), dedupe=dd)
        arr = kp_arrays(feats)
        out[f"{label}__pixels"] = px.astype(np.uint8) if np.all(px == np.rint(px)) and px.max() < 256 else px
        for k, v in arr.items():
            out[f"{label}__{k}"] = v
        meta.append(dict(label=label, alpha=a, scales=list(scales), dedupe=dd, shape=[nr, nc]))
    out["meta"] = np.array(json.dumps(meta))
    save("detector.npz", **out)
    print("detector cases", len(meta))


# --------------------------------------------------------------------------
# descriptor cases
# --------------------------------------------------------------------------

def make_descriptor():
    rng = np.random.default_rng(303)
    recs = dict(img_id=[], row=[], col=[], scale=[], beta0=[], d=[], l_max=[], orient=[], desc=[])
    images = []
    # (a) reference-test style random float images with no ramp
    for t in range(24):
        nr, nc = int(rng.integers(40, 90)), int(rng.integers(40, 90))
        images.append((rng.uniform(0, 255, size=(nr, nc)), None))
    # (b) ramped uint8 scene crops (flat regions + ramp)
    s = scenes.scene(512, 512, 11)
    for t in range(4):
        r0, c0 = int(rng.integers(0, 200)), int(rng.integers(0, 200))
        crop = s[r0:r0 + 200, c0:c0 + 260].astype(np.float64)
        images.append((crop, R_img.default_alpha(*crop.shape)))
    img_store = {}
    for iid, (px, alpha) in enumerate(images):
        if alpha is None:
            rimg = R_img.RampedImage(px, 1e-9, "t")
            img_store[f"img{iid}"] = px
        else:
            rimg = R_img.apply_linear_ramp(R_img.IntensityImage(px, "t"), alpha)
            img_store[f"img{iid}"] = px.astype(np.uint8)
            img_store[f"alpha{iid}"] = np.float64(alpha)
        nr, nc = px.shape
        n_kp = 6 if alpha is None else 40
        for _ in range(n_kp):
            row, col = int(rng.integers(0, nr)), int(rng.integers(0, nc))
            if alpha is None:
                cfg = R_desc.DescriptorConfig(beta0=0.0625, d=4, l_max=64,
                                              orientation_normalize=bool(rng.integers(0, 2)))
                scale = int(rng.choice([16, 32, 64]))
            else:
                cfg = R_desc.DescriptorConfig(beta0=0.0625, d=4, l_max=128, orientation_normalize=True)
                scale = int(rng.choice([8, 16, 32, 64, 128]))
            fp = R_det.FeaturePoint(row, col, scale, "max", 0, 0.0)
            v = R_desc.compute_descriptor(rimg, fp, cfg).values
            for k, val in (("img_id", iid), ("row", row), ("col", col), ("scale", scale),
                           ("beta0", cfg.beta0), ("d", cfg.d), ("l_max", cfg.l_max),
                           ("orient", cfg.orientation_normalize), ("desc", v)):
                recs[k].append(val)
    out = {k: np.array(v) for k, v in recs.items()}
    out.update(img_store)
    save("descriptor.npz", **out)
    print("descriptor cases", len(recs["row"]))


# --------------------------------------------------------------------------
# matcher cases
# --------------------------------------------------------------------------

def described(desc):
    feats = [R_det.FeaturePoint(i, 0, 16, "max", 0, 0.0) for i in range(len(desc))]
    return R_desc.DescribedFeatures("m", feats, np.asarray(desc, np.float64))


def make_matcher():
    rng = np.random.default_rng(77)
    out = {}
    cases = []
    # random unit-ish descriptors with planted near-copies and exact clusters
    for k, (n1, n2) in enumerate([(40, 55), (300, 280), (700, 650), (1, 1), (0, 5)]):
        A = rng.random((n1, 128)).astype(np.float32).astype(np.float64)
        A /= np.linalg.norm(A, axis=1, keepdims=True) + 1e-30
        A = A.astype(np.float32).astype(np.float64)
        B = rng.random((n2, 128)).astype(np.float32).astype(np.float64)
        if n1 and n2:
            m = min(n1, n2) // 2
            B[:m] = (A[:m] + rng.normal(0, 0.01, (m, 128))).astype(np.float32)
            if n1 > 10 and n2 > 10:
                B[m:m + 4] = A[0]  # exact duplicates of one row -> column ties
                A[5] = A[6]  # identical rows -> row ties
        cases.append((f"rand{k}", A, B))
    # real descriptors from the reference (saturated clusters, F6)
    s = scenes.scene(512, 512, 5).astype(np.float64)
    a, b = s[100:356, 0:300], s[100:356, 180:480]
    cfg = R_desc.DescriptorConfig(beta0=0.0625, d=4, l_max=64)
    sets = []
    for px in (a, b):
        r = R_img.apply_linear_ramp(R_img.IntensityImage(px, "x"), R_img.default_alpha(*px.shape))
        f = R_det.detect_features(r, R_det.ScaleSet((16, 32, 64)))
        sets.append(R_desc.describe_features(r, f, cfg).descriptors.astype(np.float32).astype(np.float64))
    cases.append(("scene", sets[0], sets[1]))
    meta = []
    for label, A, B in cases:
        out[f"{label}__A"] = A.astype(np.float32)
        out[f"{label}__B"] = B.astype(np.float32)
        for strat, ds in (("nearest_neighbor", 0.35), ("nearest_neighbor", 1.2), ("threshold_all", 0.35)):
            if strat == "threshold_all" and len(A) * len(B) > 100000:
                ds = 0.25
            pairs = R_match.match_features(described(A), described(B), R_match.MatcherConfig(ds, strat))
            tag = f"{label}__{strat}__{ds}"
            out[f"{tag}__ref1"] = np.array([p.ref1 for p in pairs], np.int64)
            out[f"{tag}__ref2"] = np.array([p.ref2 for p in pairs], np.int64)
            out[f"{tag}__delta"] = np.array([p.delta for p in pairs], np.float64)
            meta.append(dict(label=label, strategy=strat, delta_s=ds, tag=tag, n=len(pairs)))
    out["meta"] = np.array(json.dumps(meta))
    save("matcher.npz", **out)
    print("matcher cases", len(meta))


# --------------------------------------------------------------------------
# RANSAC / rigid estimation cases, plus the scalar-call sample stream
# --------------------------------------------------------------------------

def pairs_from_xy(src, dst):
    return [R_match.MatchPair((float(sy), float(sx)), (float(dy), float(dx)), 0.0, i, i)
            for i, ((sx, sy), (dx, dy)) in enumerate(zip(src, dst))]


def make_ransac():
    rng = np.random.default_rng(99)
    out = {}
    meta = []
    cases = []
    for k in range(10):
        th = float(rng.uniform(-0.4, 0.4)) if k % 3 else 0.0
        truth = R_reg.RigidTransform(th, float(rng.uniform(-60, 60)), float(rng.uniform(-60, 60)))
        n_in, n_out = int(rng.integers(8, 300)), int(rng.integers(0, 200))
        src_in = rng.integers(0, 800, size=(n_in, 2)).astype(np.float64)  # integer pixel coords
        dst_in = truth.transform_points(src_in)
        if k % 2:
            dst_in = np.rint(dst_in)
        src = np.vstack([src_in, rng.integers(0, 800, size=(n_out, 2))]).astype(np.float64)
        dst = np.vstack([dst_in, rng.integers(0, 800, size=(n_out, 2))]).astype(np.float64)
        perm = rng.permutation(len(src))
        cases.append((f"syn{k}", src[perm], dst[perm], dict(iterations=int(rng.choice([200, 1000, 2000])),
                                                           inlier_tol=3.0, min_inliers=8, seed=int(k * 7 + 1))))
    # pure noise -> RegistrationError
    cases.append(("noise", rng.uniform(0, 400, (30, 2)), rng.uniform(0, 400, (30, 2)),
                  dict(iterations=500, inlier_tol=1.0, min_inliers=8, seed=2)))
    # too few pairs
    cases.append(("few", np.arange(10.0).reshape(5, 2), np.arange(10.0).reshape(5, 2) + 1,
                  dict(iterations=100, inlier_tol=3.0, min_inliers=8, seed=0)))
    # degenerate-heavy: many coincident source points
    src = np.repeat(np.array([[5.0, 5.0], [100.0, 40.0]]), 20, axis=0)
    cases.append(("degenerate", src, src + np.array([3.0, -2.0]),
                  dict(iterations=300, inlier_tol=3.0, min_inliers=8, seed=4)))
    for label, src, dst, cfgd in cases:
        cfg = R_reg.RansacConfig(**cfgd)
        try:
            res = R_reg.ransac_rigid(pairs_from_xy(src, dst), cfg)
            ok = True
            model = np.array([res.transform.theta, res.transform.t_x, res.transform.t_y])
            inl = np.array(res.inliers, np.int64)
            rms, cons = res.residual_rms, res.consensus_size
        except RegistrationError:
            ok, model, inl, rms, cons = False, np.zeros(3), np.zeros(0, np.int64), 0.0, 0
        out[f"{label}__src"], out[f"{label}__dst"] = src, dst
        out[f"{label}__model"], out[f"{label}__inliers"] = model, inl
        out[f"{label}__rms"], out[f"{label}__consensus"], out[f"{label}__ok"] = rms, cons, ok
        meta.append(dict(label=label, **cfgd))
    # estimate_rigid KATs on random point sets (refit path: column means, pairwise sums)
    est = []
    for k in range(20):
        m = int(rng.integers(2, 400))
        s_ = rng.integers(0, 1000, size=(m, 2)).astype(np.float64)
        d_ = s_ @ np.array([[0.9, -0.3], [0.3, 0.9]]) + rng.normal(0, 2, (m, 2))
        t = R_reg.estimate_rigid(s_, d_)
        out[f"est{k}__src"], out[f"est{k}__dst"] = s_, d_
        out[f"est{k}__model"] = np.array([t.theta, t.t_x, t.t_y])
        est.append(k)
    # scalar-call sample streams (registration.py:164, 170-173)
    streams = []
    for seed in (0, 1, 11, 99, 12345, 2**40 + 3):
        for n in (2, 3, 17, 1242, 50000):
            r = np.random.default_rng(seed)
            v = []
            for _ in range(300):
                i = int(r.integers(0, n))
                j = int(r.integers(0, n - 1))
                if j >= i:
                    j += 1
                v.append((i, j))
            out[f"stream_{seed}_{n}"] = np.array(v, np.int64)
            streams.append([seed, n])
    out["meta"] = np.array(json.dumps(dict(cases=meta, est=est, streams=streams)))
    save("ransac.npz", **out)
    print("ransac cases", len(meta))


# --------------------------------------------------------------------------
# end-to-end small pair through the whole reference chain
# --------------------------------------------------------------------------

def make_e2e():
    s = scenes.scene(640, 640, 3)
    a, b = s[100:484, 0:400], s[100:484, 180:580]  # 384x400 crops, integer shift
    out = dict(a=a, b=b)
    cfg = R_desc.DescriptorConfig(beta0=0.0625, d=4, l_max=64)
    described_sets = []
    for tag, px in (("a", a), ("b", b)):
        pxf = px.astype(np.float64)
        r = R_img.apply_linear_ramp(R_img.IntensityImage(pxf, tag), R_img.default_alpha(*px.shape))
        feats = R_det.detect_features(r, R_det.ScaleSet((16, 32, 64)))
        ds = R_desc.describe_features(r, feats, cfg)
        for k, v in kp_arrays(feats).items():
            out[f"{tag}__{k}"] = v
        out[f"{tag}__desc"] = ds.descriptors
        described_sets.append(ds)
    # P3 convention: match on the fp32-rounded descriptors
    d32 = [R_desc.DescribedFeatures(x.image_id, x.features, x.descriptors.astype(np.float32).astype(np.float64))
           for x in described_sets]
    pairs = R_match.match_features(d32[0], d32[1], R_match.MatcherConfig())
    out["m__ref1"] = np.array([p.ref1 for p in pairs], np.int64)
    out["m__ref2"] = np.array([p.ref2 for p in pairs], np.int64)
    out["m__delta"] = np.array([p.delta for p in pairs])
    res = R_reg.ransac_rigid(pairs, R_reg.RansacConfig(iterations=1000, inlier_tol=3.0, min_inliers=8, seed=0))
    out["r__model"] = np.array([res.transform.theta, res.transform.t_x, res.transform.t_y])
    out["r__inliers"] = np.array(res.inliers, np.int64)
    out["r__rms"], out["r__consensus"] = res.residual_rms, res.consensus_size
    save("e2e.npz", **out)
    print("e2e matches", len(pairs), "inliers", len(res.inliers))


def compositor_cases():
    """(label, [(image, theta, tx, ty)], blend, resample) -- seeded."""
    rng = np.random.default_rng(2405)
    cases = []
    f = lambda h, w: rng.uniform(0, 255, size=(h, w))  # noqa: E731
    u = lambda h, w: rng.integers(0, 256, size=(h, w)).astype(np.uint8)  # noqa: E731
    cases.append(("identity_bilinear", [(f(40, 60), 0.0, 0.0, 0.0)], "feather", "bilinear"))
    cases.append(("identity_nearest", [(f(33, 29), 0.0, 0.0, 0.0)], "feather", "nearest"))
    cases.append(("offset_pair", [(f(30, 50), 0.0, 0.0, 0.0), (f(30, 50), 0.0, 20.0, 0.0)], "feather", "bilinear"))
    cases.append(("negative_offset", [(f(40, 40), 0.0, 0.0, 0.0), (f(40, 40), 0.0, -13.0, -7.0)], "feather",
                  "bilinear"))
    cases.append(("rotated_trio_u8", [(u(48, 64), 0.0, 0.0, 0.0), (u(48, 64), math.radians(3.0), 30.25, -4.75),
                                      (u(40, 56), math.radians(-7.0), -11.5, 17.125)], "feather", "bilinear"))
    cases.append(("rotated_trio_nearest", [(f(48, 64), 0.0, 0.0, 0.0), (f(48, 64), math.radians(5.0), 20.5, 3.5),
                                           (f(40, 56), math.radians(-2.0), -9.0, 12.0)], "feather", "nearest"))
    cases.append(("overwrite_rot", [(f(36, 52), 0.0, 0.0, 0.0), (f(36, 52), math.radians(11.0), 14.0, -6.0)],
                  "overwrite", "bilinear"))
    cases.append(("overwrite_nearest_u8", [(u(36, 52), 0.3, 5.0, 5.0), (u(30, 44), -0.2, 20.0, -3.0)],
                  "overwrite", "nearest"))
    cases.append(("half_turn", [(f(25, 31), 0.0, 0.0, 0.0), (f(25, 31), math.pi, 40.0, 30.0)], "feather",
                  "bilinear"))
    src = scenes.scene(120, 200, 4).astype(np.float64)
    cases.append(("crop_restitch", [(src[:, :120], 0.0, 0.0, 0.0), (src[:, 60:], 0.0, 60.0, 0.0)], "feather",
                  "bilinear"))
    cases.append(("quarter_turn", [(f(50, 50), 0.0, 0.0, 0.0), (f(50, 50), math.pi / 2, 50.0, 0.0)], "feather",
                  "bilinear"))
    return cases


def make_compositor():
    from peakstitch import compositor as R_comp

    out, meta = {}, []
    for label, items, blend, resample in compositor_cases():
        ids = [f"i{k}" for k in range(len(items))]
        placements = [R_comp.Placement(i, R_reg.RigidTransform(th, tx, ty)) for i, (_, th, tx, ty) in zip(ids, items)]
        dims = {i: it[0].shape for i, it in zip(ids, items)}
        canvas = R_comp.compute_canvas(placements, dims)
        pix = R_comp.warp_and_blend({i: it[0] for i, it in zip(ids, items)}, placements, canvas, blend=blend,
                                    resample=resample)
        for k, it in enumerate(items):
            out[f"{label}__img{k}"] = it[0]
        out[f"{label}__pixels"] = pix
        out[f"{label}__weightmap"] = canvas.weightmap
        meta.append(dict(label=label, blend=blend, resample=resample,
                         transforms=[[float(th), float(tx), float(ty)] for (_, th, tx, ty) in items],
                         canvas=[canvas.width, canvas.height, *canvas.origin_offset]))
    save("compositor.npz", meta=json.dumps(meta), **out)


# --------------------------------------------------------------------------
# per-pair outcomes of the reference chain at config size (C1, C3, C5):
# keypoints exact, success flags equal, match-set
# differences classified by the REFERENCE's own row / column distance gaps
# --------------------------------------------------------------------------

TAU_KEEP = 2.5e-7  # gaps below this are stored (covers the fp32 and fp64 chains' classification)


def _ref_prepare(args):
    px, wmin, wmax = args
    from peakstitch import pipeline as R_pipe

    cfg = R_pipe.PipelineConfig(window_min=wmin, window_max=wmax)
    p = R_pipe.prepare_image(R_img.IntensityImage(px.astype(np.float64), "x"), cfg)
    return kp_arrays(p.described.features), p.described.descriptors


def _gaps(dist, axis):
    """second-smallest minus smallest along ``axis`` (0 on exact ties)."""
    part = np.partition(dist, 1, axis=axis)
    lo = np.take(part, 0, axis=axis)
    hi = np.take(part, 1, axis=axis) if dist.shape[axis] > 1 else np.full_like(lo, np.inf)
    return hi - lo


def _ref_pair(args):
    """The reference's register_prepared on one pair (match_features + ransac_rigid),
    plus the near-tie structure of ITS distance matrix (captured from the
    reference's own _distance_matrix call, not recomputed)."""
    desc_a, kp_a, desc_b, kp_b, iters, seed, delta_s = args
    cap = {}
    orig = R_match._distance_matrix

    def capture(a, b):
        cap["d"] = orig(a, b)
        return cap["d"]

    R_match._distance_matrix = capture
    try:
        fa = [R_det.FeaturePoint(int(r), int(c), 0, "max", 0, 0.0) for r, c in zip(kp_a["row"], kp_a["col"])]
        fb = [R_det.FeaturePoint(int(r), int(c), 0, "max", 0, 0.0) for r, c in zip(kp_b["row"], kp_b["col"])]
        pairs = R_match.match_features(R_desc.DescribedFeatures("a", fa, desc_a), R_desc.DescribedFeatures("b", fb, desc_b),
                                       R_match.MatcherConfig(delta_s))
    finally:
        R_match._distance_matrix = orig
    d = cap["d"]
    rg, cg = _gaps(d, 1), _gaps(d, 0)
    out = dict(ref1=np.array([p.ref1 for p in pairs], np.int32), ref2=np.array([p.ref2 for p in pairs], np.int32),
               delta=np.array([p.delta for p in pairs], np.float64))
    near_r = np.flatnonzero(rg < TAU_KEEP)
    near_c = np.flatnonzero(cg < TAU_KEEP)
    out.update(near_rows=near_r.astype(np.int32), near_rows_gap=rg[near_r],
               near_cols=near_c.astype(np.int32), near_cols_gap=cg[near_c])
    try:
        res = R_reg.ransac_rigid(pairs, R_reg.RansacConfig(iterations=iters, inlier_tol=3.0, min_inliers=8, seed=seed))
        out.update(ok=True, inliers=np.array(res.inliers, np.int32), consensus=res.consensus_size,
                   model=np.array([res.transform.theta, res.transform.t_x, res.transform.t_y]), rms=res.residual_rms)
    except RegistrationError:
        out.update(ok=False, inliers=np.zeros(0, np.int32), consensus=0, model=np.zeros(3), rms=0.0)
    return out


def make_pairs(which=("c1", "c3", "c5")):
    """C1 (1 pair), C3 (all 36 pairs of the nine crops, per-pair seeds
    _pair_seed(0, a, b), mosaic.py:75-76) and C5 (pairs 0..7, RGB -> the
    reference's to_grayscale).  Keypoints, matches, RANSAC outcome and the
    near-tie rows / columns of every pair go to tests/golden/pairs_<cfg>.npz."""
    import multiprocessing as mp
    from peakstitch import mosaic as R_mosaic

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    procs = min(8, os.cpu_count() or 1)
    for cfgname in which:
        t0 = time.time()
        if cfgname == "c1":
            a, b = scenes.config1_pair(0)
            grey, wmin, wmax, iters = [a, b], 16, 64, 1000
            jobs = [(0, 1, 0)]
        elif cfgname == "c3":
            imgs, _ = scenes.config3_images(0)
            grey, wmin, wmax, iters = imgs, 32, 128, 2000
            jobs = [(x, y, R_mosaic._pair_seed(0, x, y)) for x in range(9) for y in range(x + 1, 9)]
        else:
            grey = []
            for p in range(8):
                i1, i2, _ = scenes.config5_pair(p)
                grey += [R_img.to_grayscale(i1), R_img.to_grayscale(i2)]
            wmin, wmax, iters = 16, 64, 2000
            jobs = [(2 * p, 2 * p + 1, 0) for p in range(8)]
        with mp.get_context("fork").Pool(procs) as pool:
            prepared = pool.map(_ref_prepare, [(g, wmin, wmax) for g in grey])
            outs = pool.map(_ref_pair, [(prepared[x][1], prepared[x][0], prepared[y][1], prepared[y][0], iters,
                                         seed, 0.35) for x, y, seed in jobs], chunksize=1)
        out = {}
        for k, (kp, _) in enumerate(prepared):
            for f in ("row", "col", "value"):
                out[f"img{k}__{f}"] = kp[f]
        meta = []
        for q, ((x, y, seed), o) in enumerate(zip(jobs, outs)):
            for f, v in o.items():
                out[f"pair{q}__{f}"] = np.asarray(v)
            meta.append(dict(a=x, b=y, seed=int(seed), ok=bool(o["ok"]), n_matches=int(len(o["ref1"])),
                             consensus=int(o["consensus"])))
        if cfgname == "c5":  # the RGB inputs are regenerated from scenes.config5_pair on the box
            out["grey_digest"] = np.array([scenes.scene_digest(g.view(np.uint8)) for g in grey])
        out["meta"] = np.array(json.dumps(dict(config=cfgname, window=[wmin, wmax], iterations=iters,
                                               tau_keep=TAU_KEEP, pairs=meta)))
        save(f"pairs_{cfgname}.npz", **out)
        print(cfgname, "pairs", len(jobs), "ok", sum(m["ok"] for m in meta), "%.0fs" % (time.time() - t0))


def make_scene_digests():
    d = {}
    for (h, w, seed) in [(64, 96, 0), (256, 256, 1), (512, 512, 7), (1600, 2688, 0), (2048, 2048, 0)]:
        d[f"{h}x{w}_seed{seed}"] = scenes.scene_digest(scenes.scene(h, w, seed))
    with open(os.path.join(HERE, "scene_digests.json"), "w") as f:
        json.dump(d, f, indent=1)


if __name__ == "__main__":
    t = time.time()
    what = sys.argv[1:] or ["detector", "descriptor", "matcher", "ransac", "e2e", "compositor", "digests"]
    for w in what:
        {"detector": make_detector, "descriptor": make_descriptor, "matcher": make_matcher,
         "ransac": make_ransac, "e2e": make_e2e, "compositor": make_compositor,
         "digests": make_scene_digests, "pairs": make_pairs,
         "pairs_c1": lambda: make_pairs(("c1",)), "pairs_c3": lambda: make_pairs(("c3",)),
         "pairs_c5": lambda: make_pairs(("c5",))}[w]()
    env = dict(numpy=np.__version__, python=sys.version.split()[0])
    with open(os.path.join(HERE, "ENV.json"), "w") as f:
        json.dump(env, f)
    print("done in %.1fs" % (time.time() - t))
