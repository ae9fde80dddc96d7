"""CPU oracle for the LP-SIFT hot path: detect -> describe -> match -> RANSAC.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline leg may import this module, and only as the
checker / the timed CPU port.  The product package
(``paper_2405_08578_b200``) never imports it and has no CPU fallback.

This is an independent numpy restatement of the reference package
``peakstitch`` (``/root/reference/pkg/src/peakstitch``), written so that the
float64 results are bit-identical to the reference on the same host: every
reduction uses the same numpy reduction (and therefore the same summation
order) as the reference, and every libm call is the same one.  Each function
cites the reference lines it restates.

Pinning: ``tests/golden/make_golden.py`` runs the real reference (importable
in the build container) on seeded inputs and commits its outputs under
``tests/golden/``; ``tests/test_oracle_golden.py`` checks this module against
those fixtures (bit-exact keypoints / matches / inlier sets, descriptors to
1e-12).  The parity of the sample stream (numpy PCG64) is pinned the same way.
"""

from __future__ import annotations

import math

import numpy as np

TWO_PI = 2.0 * math.pi  # descriptor.py:31
MIN_WINDOW = 8  # detector.py:20
RAMP_SPAN_LIMIT = 0.05 * 255.0  # imaging.py:24

POL_MAX = 0  # "max" sorts before "min" (detector.py:171, string order)
POL_MIN = 1

KP_DTYPE = np.dtype(
    [("row", np.int64), ("col", np.int64), ("scale", np.int64),
     ("pol", np.int8), ("window", np.int64), ("value", np.float64)]
)


class OracleConfigError(ValueError):
    pass


# ---------------------------------------------------------------------------
# imaging.py:108-132 -- ramp
# ---------------------------------------------------------------------------

def default_alpha(nr: int, nc: int) -> float:
    """imaging.py:108-111."""
    return 1e-6 * 255.0 / (nr * nc)


def ramp(pixels: np.ndarray, alpha: float) -> np.ndarray:
    """P = I + fl(k * alpha), k = r*nc + c + 1 (imaging.py:113-132)."""
    if not math.isfinite(alpha) or alpha <= 0:
        raise OracleConfigError("alpha must be positive")
    nr, nc = pixels.shape
    if alpha * nr * nc > RAMP_SPAN_LIMIT:
        raise OracleConfigError("ramp span too large")
    k = np.arange(1, nr * nc + 1, dtype=np.float64).reshape(nr, nc)
    return np.asarray(pixels, dtype=np.float64) + k * alpha


# ---------------------------------------------------------------------------
# detector.py:20-172 -- scales, windows, extrema, dedupe, order
# ---------------------------------------------------------------------------

def scales_from_range(l_min: int, l_max: int) -> tuple[int, ...]:
    """ScaleSet.from_range (detector.py:50-61)."""
    if l_min > l_max:
        raise OracleConfigError("empty range")
    out, s = [], int(l_min)
    while s < l_max:
        out.append(s)
        s *= 2
    out.append(int(l_max))
    return tuple(out)


def check_scales(sizes, nr: int, nc: int) -> None:
    """ScaleSet.__post_init__ / validate_for (detector.py:33-68)."""
    if not sizes:
        raise OracleConfigError("empty scale set")
    if any(int(s) != s or s < MIN_WINDOW for s in sizes):
        raise OracleConfigError("window sizes must be integers >= 8")
    if any(b <= a for a, b in zip(sizes, sizes[1:])):
        raise OracleConfigError("not increasing")
    if sizes[-1] > min(nr, nc):
        raise OracleConfigError("largest window exceeds image")


def window_extrema(P: np.ndarray, L: int) -> tuple[np.ndarray, np.ndarray]:
    """Flat image indices of every L-window's first argmax / first argmin.

    Windows are row-major, trailing ones shrunk (detector.py:87-103);
    per window ``np.argmax``/``np.argmin`` on the row-major flattened window
    (detector.py:114-119).  Padding the shrunk windows with -inf/+inf keeps
    the row-major first-occurrence rule.
    """
    nr, nc = P.shape
    wr, wc = -(-nr // L), -(-nc // L)
    out = []
    for fill, fn in ((-np.inf, np.argmax), (np.inf, np.argmin)):
        pad = np.full((wr * L, wc * L), fill)
        pad[:nr, :nc] = P
        blocks = pad.reshape(wr, L, wc, L).transpose(0, 2, 1, 3).reshape(wr * wc, L * L)
        loc = fn(blocks, axis=1)
        lr, lc = loc // L, loc % L
        win = np.arange(wr * wc)
        rows = (win // wc) * L + lr
        cols = (win % wc) * L + lc
        out.append(rows * nc + cols)
    return out[0], out[1]


def detect(P: np.ndarray, sizes, dedupe: bool = True) -> np.ndarray:
    """detect_features (detector.py:154-172) -> structured KP_DTYPE array.

    Raw order is (scale ascending, window, max-then-min); dedupe keeps the
    first occurrence of each (row, col, polarity) (detector.py:139-151), which
    is the smallest scale; the final sort key (scale, window, polarity) is the
    raw order itself.
    """
    P = np.asarray(P, dtype=np.float64)
    nr, nc = P.shape
    sizes = tuple(int(s) for s in sizes)
    check_scales(sizes, nr, nc)
    parts = []
    for L in sizes:
        imax, imin = window_extrema(P, L)
        nw = imax.shape[0]
        rec = np.empty(2 * nw, dtype=KP_DTYPE)
        flat = np.empty(2 * nw, dtype=np.int64)
        flat[0::2], flat[1::2] = imax, imin
        rec["row"], rec["col"] = flat // nc, flat % nc
        rec["scale"] = L
        rec["pol"][0::2], rec["pol"][1::2] = POL_MAX, POL_MIN
        rec["window"] = np.repeat(np.arange(nw), 2)
        rec["value"] = P.ravel()[flat]
        parts.append(rec)
    raw = np.concatenate(parts)
    if not dedupe:
        return raw
    key = (raw["row"] * nc + raw["col"]) * 2 + raw["pol"]
    _, first = np.unique(key, return_index=True)
    keep = np.zeros(raw.shape[0], dtype=bool)
    keep[first] = True
    return raw[keep]


# ---------------------------------------------------------------------------
# descriptor.py:82-269 -- region geometry, gradients, orientation, histogram
# ---------------------------------------------------------------------------

def region_side(scale: int, beta0: float, d: int, l_max: int) -> int:
    """region_size (descriptor.py:82-95)."""
    if scale > l_max:
        raise OracleConfigError("scale exceeds l_max")
    beta = beta0 * (scale / l_max) ** -0.5
    w = int(math.floor(beta * scale * d + 0.5))
    w = min(w, scale)
    w -= w % d
    return max(w, d)


def fit_region(nr, nc, row, col, w, d):
    """_fit_region (descriptor.py:118-131)."""
    cap = min(nr, nc) - 2
    if cap < d:
        raise ValueError("image too small")
    if w > cap:
        w = cap - cap % d
    r0 = min(max(row - w // 2, 1), nr - 1 - w)
    c0 = min(max(col - w // 2, 1), nc - 1 - w)
    return r0, c0, w


def _axis_gradients(P, r0, c0, w):
    """Central differences over the axis region (descriptor.py:134-139)."""
    rows = slice(r0, r0 + w)
    cols = slice(c0, c0 + w)
    ga = P[r0 + 1:r0 + w + 1, cols] - P[r0 - 1:r0 + w - 1, cols]
    gb = P[rows, c0 + 1:c0 + w + 1] - P[rows, c0 - 1:c0 + w - 1]
    return np.hypot(ga, gb), np.mod(np.arctan2(gb, ga), TWO_PI)


def peak_bin(mag, ori) -> int:
    """First argmax of the 36-bin magnitude histogram (descriptor.py:142-146)."""
    k = np.minimum((ori * (36 / TWO_PI)).astype(np.intp), 35)
    hist = np.zeros(36)
    np.add.at(hist, k.ravel(), mag.ravel())  # sequential, raster order
    return int(np.argmax(hist))


def _rotated_samples(P, cy, cx, w, theta0):
    """Rotated-grid bilinear gradient samples (descriptor.py:164-216)."""
    nr, nc = P.shape
    off = np.arange(w, dtype=np.float64) - (w - 1) / 2.0
    ct, st = math.cos(-theta0), math.sin(-theta0)
    u, v = off[None, :], off[:, None]
    x = cx + ct * u - st * v
    y = cy + st * u + ct * v
    inside = (x >= 1) & (x <= nc - 2) & (y >= 1) & (y <= nr - 2)
    pr0 = max(int(np.floor(y.min())), 1)
    pr1 = min(int(np.ceil(y.max())), nr - 2)
    pc0 = max(int(np.floor(x.min())), 1)
    pc1 = min(int(np.ceil(x.max())), nc - 2)
    fa = P[pr0 + 1:pr1 + 2, pc0:pc1 + 1] - P[pr0 - 1:pr1, pc0:pc1 + 1]
    fb = P[pr0:pr1 + 1, pc0 + 1:pc1 + 2] - P[pr0:pr1 + 1, pc0 - 1:pc1]
    lx = np.clip(x, pc0, pc1) - pc0
    ly = np.clip(y, pr0, pr1) - pr0
    ix0 = np.minimum(np.floor(lx).astype(np.intp), max(pc1 - pc0 - 1, 0))
    iy0 = np.minimum(np.floor(ly).astype(np.intp), max(pr1 - pr0 - 1, 0))
    tx, ty = lx - ix0, ly - iy0
    ix1 = np.minimum(ix0 + 1, pc1 - pc0)
    iy1 = np.minimum(iy0 + 1, pr1 - pr0)
    sx, sy = 1.0 - tx, 1.0 - ty

    def bil(f):
        return (f[iy0, ix0] * sy * sx + f[iy0, ix1] * sy * tx
                + f[iy1, ix0] * ty * sx + f[iy1, ix1] * ty * tx)

    a_s, b_s = bil(fa), bil(fb)
    return np.hypot(a_s, b_s) * inside, np.mod(np.arctan2(b_s, a_s) - theta0, TWO_PI)


def describe_one(P, row, col, scale, beta0=0.0625, d=4, l_max=128, orient=True):
    """compute_descriptor (descriptor.py:219-256) -> float64 (d*d*8,)."""
    nr, nc = P.shape
    w = region_side(scale, beta0, d, l_max)
    r0, c0, w = fit_region(nr, nc, row, col, w, d)
    ws = w // d
    if orient:
        k = peak_bin(*_axis_gradients(P, r0, c0, w))
        theta0 = (k + 0.5) * (TWO_PI / 36)
        h = (w - 1) / 2.0
        cy = min(max(float(row), 1.0 + h), (nr - 2.0) - h)
        cx = min(max(float(col), 1.0 + h), (nc - 2.0) - h)
        mag, ori = _rotated_samples(P, cy, cx, w, theta0)
    else:
        mag, ori = _axis_gradients(P, r0, c0, w)
    ob = np.minimum((ori * (8 / TWO_PI)).astype(np.intp), 7)
    cell_of = np.arange(w) // ws
    idx = (cell_of[:, None] * d + cell_of[None, :]) * 8 + ob
    vec = np.zeros(d * d * 8)
    np.add.at(vec, idx.ravel(), mag.ravel())
    n = math.sqrt(float(np.dot(vec, vec)))
    if n > 0.0:
        vec /= n
        np.minimum(vec, 0.2, out=vec)
        vec /= math.sqrt(float(np.dot(vec, vec)))
    return vec


def describe(P, kps, beta0=0.0625, d=4, l_max=128, orient=True) -> np.ndarray:
    """describe_features (descriptor.py:259-269)."""
    out = np.zeros((len(kps), d * d * 8))
    for i in range(len(kps)):
        out[i] = describe_one(P, int(kps["row"][i]), int(kps["col"][i]),
                              int(kps["scale"][i]), beta0, d, l_max, orient)
    return out


# ---------------------------------------------------------------------------
# matcher.py:48-95 -- exact float64 distances, MNN / threshold_all, order
# ---------------------------------------------------------------------------

def distances(A: np.ndarray, B: np.ndarray, chunk: int = 32):
    """Yield (i0, dist[i0:i1, :]) with the reference's bits.

    matcher.py:48-54 uses ``np.linalg.norm(b - a[i], axis=1)``, i.e. a
    contiguous last-axis add.reduce of squares (numpy pairwise summation),
    then sqrt; the same reduction is applied here chunk-wise.
    """
    A = np.asarray(A, np.float64)
    B = np.asarray(B, np.float64)
    for i0 in range(0, A.shape[0], chunk):
        diff = B[None, :, :] - A[i0:i0 + chunk, None, :]
        yield i0, np.sqrt(np.add.reduce(diff * diff, axis=2))


def match(A, B, delta_s: float = 0.35, strategy: str = "nearest_neighbor"):
    """match_features (matcher.py:57-95) -> (ref1, ref2, delta) sorted.

    ``strategy="ratio_test"`` is the EXTRA Lowe-ratio strategy the reference
    does not have: ``delta_s`` is the ratio r, and row i keeps
    its first nearest neighbour j when d1 < r * d2 (float64), d2 the row's
    second-smallest distance (a duplicate of the best counts; inf when B has
    one row).  Its own oracle, not pinned by the reference.
    """
    n1, n2 = len(A), len(B)
    if n1 == 0 or n2 == 0:
        e = np.zeros(0, np.int64)
        return e, e.copy(), np.zeros(0)
    r1, r2, dl = [], [], []
    if strategy == "ratio_test":
        for i0, D in distances(A, B):
            j = np.argmin(D, axis=1)
            rows = np.arange(D.shape[0])
            d1 = D[rows, j]
            d2 = np.partition(D, 1, axis=1)[:, 1] if n2 > 1 else np.full(D.shape[0], np.inf)
            ok = d1 < delta_s * d2
            r1.append(rows[ok] + i0), r2.append(j[ok]), dl.append(d1[ok])
    elif strategy == "threshold_all":
        for i0, D in distances(A, B):
            ii, jj = np.nonzero(D < delta_s)  # row-major, like np.argwhere
            r1.append(ii + i0), r2.append(jj), dl.append(D[ii, jj])
    else:
        nn12 = np.empty(n1, np.int64)
        best12 = np.empty(n1)
        col_best = np.full(n2, np.inf)
        col_arg = np.zeros(n2, np.int64)
        for i0, D in distances(A, B):
            j = np.argmin(D, axis=1)
            nn12[i0:i0 + D.shape[0]] = j
            best12[i0:i0 + D.shape[0]] = D[np.arange(D.shape[0]), j]
            ci = np.argmin(D, axis=0)
            cv = D[ci, np.arange(n2)]
            upd = cv < col_best  # strict: earlier rows win ties (first argmin)
            col_best[upd] = cv[upd]
            col_arg[upd] = ci[upd] + i0
        rows = np.arange(n1)
        ok = (col_arg[nn12] == rows) & (best12 < delta_s)
        r1.append(rows[ok]), r2.append(nn12[ok]), dl.append(best12[ok])
    ref1 = np.concatenate(r1).astype(np.int64)
    ref2 = np.concatenate(r2).astype(np.int64)
    delta = np.concatenate(dl)
    order = np.lexsort((ref2, ref1, delta))
    return ref1[order], ref2[order], delta[order]


# ---------------------------------------------------------------------------
# registration.py:27-203 -- rigid model, 2-point RANSAC
# ---------------------------------------------------------------------------

def norm_theta(theta: float) -> float:
    """RigidTransform.__post_init__ (registration.py:33-38)."""
    t = math.remainder(theta, 2.0 * math.pi)
    if t <= -math.pi:
        t += 2.0 * math.pi
    return t


class Degenerate(ValueError):
    pass


class NoConsensus(RuntimeError):
    pass


def fit_rigid(src: np.ndarray, dst: np.ndarray):
    """estimate_rigid (registration.py:107-131) -> normalised (theta, tx, ty).

    numpy's orders: mean(axis=0) of an (m, 2) array is a sequential column
    sum / m; ``(s*d).sum()`` is a pairwise sum over the flattened 2m
    products; the cross term is a 1-D pairwise sum.
    """
    src = np.asarray(src, np.float64)
    dst = np.asarray(dst, np.float64)
    if src.shape != dst.shape or src.ndim != 2 or src.shape[1] != 2 or src.shape[0] < 2:
        raise Degenerate("bad shapes")
    cs, cd = src.mean(axis=0), dst.mean(axis=0)
    s, t = src - cs, dst - cd
    if not (np.abs(s) > 1e-12).any():
        raise Degenerate("coincident")
    dot = float((s * t).sum())
    cross = float((s[:, 0] * t[:, 1] - s[:, 1] * t[:, 0]).sum())
    th = math.atan2(cross, dot)
    c, si = math.cos(th), math.sin(th)
    tx = cd[0] - (c * cs[0] - si * cs[1])
    ty = cd[1] - (si * cs[0] + c * cs[1])
    return norm_theta(th), float(tx), float(ty)


def residuals(model, src, dst) -> np.ndarray:
    """transfer_errors (registration.py:66-73, 134-140)."""
    th, tx, ty = model
    c, s = math.cos(th), math.sin(th)
    px = c * src[:, 0] - s * src[:, 1] + tx
    py = s * src[:, 0] + c * src[:, 1] + ty
    return np.hypot(dst[:, 0] - px, dst[:, 1] - py)


def sample_stream(seed: int, n: int, iterations: int) -> np.ndarray:
    """(iterations, 2) sample indices of registration.py:164, 170-173.

    One vector draw with highs [n, n-1, n, n-1, ...] reproduces the
    reference's alternating scalar ``rng.integers`` calls (SURVEY.md F8,
    re-checked in tests/test_oracle_golden.py).
    """
    rng = np.random.default_rng(seed)
    highs = np.tile(np.array([n, n - 1], dtype=np.int64), iterations)
    v = rng.integers(0, highs).reshape(iterations, 2)
    v[:, 1] += v[:, 1] >= v[:, 0]
    return v


def ransac(src, dst, iterations=2000, tol=3.0, min_inliers=8, seed=0):
    """ransac_rigid (registration.py:149-203).

    Returns dict(model=(theta, tx, ty), inliers, rms, consensus).  Raises
    NoConsensus where the reference raises RegistrationError.
    """
    src = np.asarray(src, np.float64)
    dst = np.asarray(dst, np.float64)
    n = src.shape[0]
    if n < min_inliers:
        raise NoConsensus("too few pairs")
    samples = sample_stream(seed, n, iterations)
    best = (0, math.inf, None)
    for i, j in samples:
        try:
            model = fit_rigid(src[[i, j]], dst[[i, j]])
        except Degenerate:
            continue
        e = residuals(model, src, dst)
        m = e <= tol
        cnt = int(m.sum())
        if cnt == 0 or cnt < best[0]:
            continue
        rms = float(np.sqrt(np.mean(e[m] ** 2)))
        if cnt > best[0] or rms < best[1]:
            best = (cnt, rms, m)
    if best[2] is None or best[0] < min_inliers:
        raise NoConsensus("consensus below min_inliers")
    model = fit_rigid(src[best[2]], dst[best[2]])
    e = residuals(model, src, dst)
    fm = e <= tol
    if int(fm.sum()) < min_inliers:
        raise NoConsensus("refit lost consensus")
    return dict(model=model, inliers=np.flatnonzero(fm), rms=float(np.sqrt(np.mean(e[fm] ** 2))),
                consensus=best[0])


def pair_points(ref1, ref2, kp1, kp2):
    """_pair_points (registration.py:143-146): (x, y) = (col, row)."""
    src = np.stack([kp1["col"][ref1], kp1["row"][ref1]], axis=1).astype(np.float64)
    dst = np.stack([kp2["col"][ref2], kp2["row"][ref2]], axis=1).astype(np.float64)
    return src, dst


# ---------------------------------------------------------------------------
# compositor.py:20-160 -- canvas bounds, inverse-mapped resampling, blending
# (SURVEY.md §8(f) #2).  Transforms are (theta, t_x, t_y) triples with the
# RigidTransform semantics of registration.py:33-73.
# ---------------------------------------------------------------------------

SNAP = 1e-6  # compositor.py:20


def apply_rigid(theta: float, tx: float, ty: float, x, y):
    """RigidTransform.transform_points (registration.py:66-73): numpy order
    (c*x - s*y) + t_x, (s*x + c*y) + t_y with host-libm cos / sin."""
    theta = norm_theta(theta)
    c, s = math.cos(theta), math.sin(theta)
    return c * x - s * y + tx, s * x + c * y + ty


def invert_rigid(theta: float, tx: float, ty: float):
    """RigidTransform.inverse (registration.py:49-55)."""
    theta = norm_theta(theta)
    c, s = math.cos(theta), math.sin(theta)
    return norm_theta(-theta), -(c * tx + s * ty), -(-s * tx + c * ty)


def snapped_corners(transform, nr: int, nc: int):
    """Transformed image corners snapped to 1e-6 (compositor.py:40-41, 51, 122-123)."""
    x = np.array([0.0, nc, 0.0, nc])
    y = np.array([0.0, 0.0, nr, nr])
    cx, cy = apply_rigid(*transform, x, y)
    return np.round(cx / SNAP) * SNAP, np.round(cy / SNAP) * SNAP


def canvas_bounds(transforms, dims):
    """compute_canvas (compositor.py:44-58) -> (width, height, dx, dy)."""
    if not transforms:
        raise ValueError("need at least one placement")
    xs, ys = zip(*(snapped_corners(t, *d) for t, d in zip(transforms, dims)))
    xs, ys = np.concatenate(xs), np.concatenate(ys)
    dx, dy = math.floor(xs.min()), math.floor(ys.min())
    return math.ceil(xs.max()) - dx, math.ceil(ys.max()) - dy, dx, dy


def composite(images, transforms, bounds, blend: str = "feather", resample: str = "bilinear"):
    """warp_and_blend (compositor.py:84-160) -> (pixels, weightmap)."""
    if blend not in ("feather", "overwrite"):
        raise ValueError(f"unknown blend mode {blend!r}")
    if resample not in ("bilinear", "nearest"):
        raise ValueError(f"unknown resample mode {resample!r}")
    width, height, dx, dy = bounds
    acc = np.zeros((height, width))
    wsum = np.zeros((height, width))
    cnt = np.zeros((height, width), dtype=np.int64)
    solo = np.zeros((height, width))
    for img, t in zip(images, transforms):
        nr, nc = img.shape
        cx, cy = snapped_corners(t, nr, nc)
        r0, r1 = max(math.floor(cy.min()) - dy, 0), min(math.ceil(cy.max()) - dy, height)
        c0, c1 = max(math.floor(cx.min()) - dx, 0), min(math.ceil(cx.max()) - dx, width)
        if r0 >= r1 or c0 >= c1:
            continue
        Y, X = np.meshgrid(np.arange(r0, r1, dtype=np.float64) + dy, np.arange(c0, c1, dtype=np.float64) + dx,
                           indexing="ij")
        sx, sy = apply_rigid(*invert_rigid(*t), X, Y)
        ok = (sx >= 0) & (sx <= nc - 1) & (sy >= 0) & (sy <= nr - 1)
        xs, ys = np.clip(sx, 0, nc - 1), np.clip(sy, 0, nr - 1)
        if resample == "bilinear":  # _sample_bilinear (compositor.py:61-74)
            ix = np.clip(np.floor(xs).astype(np.int64), 0, max(nc - 2, 0))
            iy = np.clip(np.floor(ys).astype(np.int64), 0, max(nr - 2, 0))
            fx, fy = xs - ix, ys - iy
            jx, jy = np.minimum(ix + 1, nc - 1), np.minimum(iy + 1, nr - 1)
            v = (img[iy, ix] * (1.0 - fy) * (1.0 - fx) + img[iy, jx] * (1.0 - fy) * fx
                 + img[jy, ix] * fy * (1.0 - fx) + img[jy, jx] * fy * fx)
        else:  # _sample_nearest (compositor.py:77-81)
            v = img[np.clip(np.rint(ys).astype(np.int64), 0, nr - 1), np.clip(np.rint(xs).astype(np.int64), 0, nc - 1)]
            v = v.astype(np.float64)
        blk = (slice(r0, r1), slice(c0, c1))
        if blend == "overwrite":
            acc[blk][ok] = v[ok]
            wsum[blk][ok] = 1.0
            cnt[blk][ok] = 1
        else:
            w = 1.0 + np.minimum(np.minimum(sx, nc - 1 - sx), np.minimum(sy, nr - 1 - sy))
            acc[blk] += np.where(ok, w * v, 0.0)
            wsum[blk] += np.where(ok, w, 0.0)
            cnt[blk] += ok
        solo[blk][ok] = v[ok]
    out = np.zeros((height, width))
    np.divide(acc, wsum, out=out, where=wsum > 0)
    out[cnt == 1] = solo[cnt == 1]
    return out, wsum
