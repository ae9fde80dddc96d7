"""Callers of the hot path (reference pipeline.py:42-209, mosaic.py:75-112).

``prepare_image`` runs ramp -> detect -> describe on the GPU and keeps the
keypoints and float32 descriptors resident; ``register_prepared`` runs
match -> RANSAC on the GPU.  ``prepare_batch`` is the batched form used for
throughput (one detect launch and one describe launch for B images).
Config parsing, reports and compositing are out of scope.
"""

from __future__ import annotations

import functools
import math
import time
from dataclasses import dataclass, fields, replace

import numpy as np
import torch

from . import device
from .detector import features_from_arrays
from .matcher import match_tensors
from .errors import ConfigError
from .records import (STRATEGY_NEAREST, STRATEGY_RATIO, STRATEGY_THRESHOLD_ALL, DescribedFeatures, DescriptorConfig,
                      IntensityImage, MatcherConfig, MatchPair, RansacConfig, RegistrationResult, RigidTransform,
                      ScaleSet, apply_linear_ramp, default_alpha)


@dataclass(frozen=True)
class PipelineConfig:
    """pipeline.py:42-117 (hot-path fields; compositing knobs accepted, unused)."""

    alpha: float | None = None
    window_min: int = 32
    window_max: int = 128
    beta0: float = 0.0625
    d: int = 4
    orientation_normalize: bool = True
    delta_s: float = 0.35
    match_strategy: str = STRATEGY_NEAREST
    ransac_iters: int = 2000
    ransac_tol: float = 3.0
    min_inliers: int = 8
    seed: int = 0
    threads: int = 1
    blend: str = "feather"
    resample: str = "bilinear"
    match_ratio: float = 0.8  # extra "ratio_test" strategy only (not a reference field)

    def __post_init__(self):
        if self.alpha is not None and (not math.isfinite(self.alpha) or self.alpha <= 0):
            raise ConfigError(f"alpha must be positive, got {self.alpha}")
        scales = ScaleSet.from_range(self.window_min, self.window_max)
        if self.d < 1 or self.d > self.window_min:
            raise ConfigError(f"subregion grid d={self.d} must be in [1, window_min={self.window_min}]")
        bound = (1.0 / self.d) * math.sqrt(scales.sizes[0] / scales.l_max)
        if not 0 < self.beta0 <= bound:
            raise ConfigError(f"beta0={self.beta0} outside (0, {bound:.6g}] for window range "
                              f"[{self.window_min}, {self.window_max}] with d={self.d}")
        if self.delta_s <= 0:
            raise ConfigError(f"delta_s must be positive, got {self.delta_s}")
        if self.match_strategy not in (STRATEGY_NEAREST, STRATEGY_THRESHOLD_ALL, STRATEGY_RATIO):
            raise ConfigError(f"unknown match strategy {self.match_strategy!r}")
        if self.ransac_iters < 1 or self.ransac_tol <= 0 or self.min_inliers < 2:
            raise ConfigError("invalid RANSAC parameters")
        if self.threads < 1:
            raise ConfigError(f"threads must be >= 1, got {self.threads}")

    def scale_set(self) -> ScaleSet:
        return ScaleSet.from_range(self.window_min, self.window_max)

    def descriptor_config(self) -> DescriptorConfig:
        return DescriptorConfig(self.beta0, self.d, self.window_max, self.orientation_normalize)

    def matcher_config(self) -> MatcherConfig:
        return MatcherConfig(self.delta_s, self.match_strategy, self.match_ratio)

    def ransac_config(self, seed: int | None = None) -> RansacConfig:
        return RansacConfig(self.ransac_iters, self.ransac_tol, self.min_inliers, self.seed if seed is None else seed)

    def with_overrides(self, overrides: dict) -> "PipelineConfig":
        unknown = set(overrides) - {f.name for f in fields(self)}
        if unknown:
            raise ConfigError(f"unknown config keys: {sorted(unknown)}")
        return replace(self, **overrides)


@dataclass(eq=False)
class PreparedImage:
    """Device-resident features of one image (slot b of a prepared batch)."""

    image: object
    keypoints: device.Keypoints
    slot: int
    desc32: torch.Tensor  # [cap, D] float32 on the GPU (valid rows [0, count))
    detect_seconds: float
    describe_seconds: float
    _described: DescribedFeatures | None = None

    @property
    def count(self) -> int:
        return int(self.keypoints.count[self.slot].item())

    @property
    def feature_count(self) -> int:
        return self.count

    @property
    def descriptors(self) -> torch.Tensor:
        return self.desc32[: self.count]

    @property
    def described(self) -> DescribedFeatures:
        """Host view (FeaturePoints + float64 upcast of the float32 descriptors)."""
        if self._described is None:
            h = self.keypoints.image(self.slot)
            n = len(h["row"])
            if "scale" not in h:
                h["scale"] = np.full(n, self.keypoints.default_scale)
                h["polarity"] = np.arange(n) % 2
                h["window"] = np.arange(n) // 2
            feats = features_from_arrays(h)
            iid = getattr(self.image, "image_id", "")
            self._described = DescribedFeatures(iid, feats, self.descriptors.double().cpu().numpy())
        return self._described


def _raw_of(img):
    px = img.pixels if hasattr(img, "pixels") else img
    if isinstance(px, torch.Tensor):
        return px
    a = np.asarray(px)
    if a.dtype != np.uint8 and np.all((a >= 0) & (a <= 255) & (a == np.rint(a))):
        a = a.astype(np.uint8)
    return torch.from_numpy(np.ascontiguousarray(a))


def prepare_batch(images, cfg: PipelineConfig, *, stream=None, meta=False) -> list:
    """Detect + describe B same-sized images with one launch per stage."""
    imgs = list(images)
    raws = [_raw_of(im) for im in imgs]
    batch = torch.stack(raws).cuda(non_blocking=True)
    nr, nc = batch.shape[1], batch.shape[2]
    alpha = cfg.alpha if cfg.alpha is not None else default_alpha(nr, nc)
    apply_linear_ramp(IntensityImage(raws[0]), alpha)  # validation (imaging.py:121-128)
    dimg = device.as_device_images(batch, alpha)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kp = device.detect(dimg, cfg.scale_set().sizes, dedupe=True, meta=meta, stream=stream)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    d32 = device.describe(dimg, kp, cfg.descriptor_config(), stream=stream)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    B = len(imgs)
    return [PreparedImage(imgs[b], kp, b, d32[b], (t1 - t0) / B, (t2 - t1) / B) for b in range(B)]


def prepare_image(img, cfg: PipelineConfig) -> PreparedImage:
    """pipeline.py:171-186 on the GPU."""
    return prepare_batch([img], cfg, meta=True)[0]


def _pairs_host(prep_a, prep_b, r1, r2, dl) -> list:
    ka, kb = prep_a.keypoints, prep_b.keypoints
    ra, ca = ka.row[prep_a.slot].cpu().numpy(), ka.col[prep_a.slot].cpu().numpy()
    rb, cb = kb.row[prep_b.slot].cpu().numpy(), kb.col[prep_b.slot].cpu().numpy()
    r1, r2, dl = r1.cpu().numpy(), r2.cpu().numpy(), dl.cpu().numpy()
    return [MatchPair((int(ra[i]), int(ca[i])), (int(rb[j]), int(cb[j])), float(d), int(i), int(j))
            for i, j, d in zip(r1, r2, dl)]


def register_device(prep_a: PreparedImage, prep_b: PreparedImage, cfg: PipelineConfig, seed=None):
    """match -> RANSAC entirely on the GPU; returns (r1, r2, delta, RansacOutcome|None)."""
    mc = cfg.matcher_config()
    r1, r2, dl = match_tensors(prep_a.descriptors, prep_b.descriptors, mc)
    rc = cfg.ransac_config(seed)
    n = int(r1.shape[0])
    if n < rc.min_inliers:
        return r1, r2, dl, None
    ka, kb = prep_a.keypoints, prep_b.keypoints
    src, dst = device.pair_points(r1, r2, ka.row[prep_a.slot], ka.col[prep_a.slot], kb.row[prep_b.slot],
                                  kb.col[prep_b.slot])
    out = device.ransac(src, dst, rc.iterations, rc.inlier_tol, rc.min_inliers, rc.seed)
    return r1, r2, dl, out


def register_prepared(prep_a: PreparedImage, prep_b: PreparedImage, cfg: PipelineConfig, seed=None):
    """pipeline.py:189-209: (pairs, RegistrationResult | None, match_s, ransac_s)."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mc = cfg.matcher_config()
    r1, r2, dl = match_tensors(prep_a.descriptors, prep_b.descriptors, mc)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pairs = _pairs_host(prep_a, prep_b, r1, r2, dl)
    rc = cfg.ransac_config(seed)
    result = None
    if len(pairs) >= rc.min_inliers:
        ka, kb = prep_a.keypoints, prep_b.keypoints
        src, dst = device.pair_points(r1, r2, ka.row[prep_a.slot], ka.col[prep_a.slot], kb.row[prep_b.slot],
                                      kb.col[prep_b.slot])
        out = device.ransac(src, dst, rc.iterations, rc.inlier_tol, rc.min_inliers, rc.seed)
        if out.ok:
            result = RegistrationResult(RigidTransform(out.theta, out.t_x, out.t_y), out.inliers.tolist(), out.rms,
                                        out.consensus)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return pairs, result, t1 - t0, t2 - t1


@dataclass(eq=False)
class StitchResult:
    """pipeline.py:212-218."""

    success: bool
    transform: object | None
    registration: RegistrationResult | None
    composite: np.ndarray | None
    report: dict


def _compositor_pixels(img):
    """The image as the compositor samples it (IntensityImage pixels)."""
    px = img.pixels if hasattr(img, "pixels") else img
    return px if isinstance(px, torch.Tensor) else np.asarray(px)


def stitch_pair(img_a, img_b, cfg: PipelineConfig) -> StitchResult:
    """pipeline.py:232-290 on the GPU: detect + describe both images, match,
    RANSAC, and (on success) the device composite in the first image's frame."""
    from . import compositor as K

    start = time.perf_counter()
    if tuple(_compositor_pixels(img_a).shape[:2]) == tuple(_compositor_pixels(img_b).shape[:2]):
        prep_a, prep_b = prepare_batch([img_a, img_b], cfg, meta=True)
    else:
        prep_a, prep_b = prepare_image(img_a, cfg), prepare_image(img_b, cfg)
    pairs, result, match_s, ransac_s = register_prepared(prep_a, prep_b, cfg)
    stitch_s = ransac_s
    composite = None
    registration = {"theta_deg": 0.0, "t_x": 0.0, "t_y": 0.0, "inliers": 0, "pairs_in": len(pairs),
                    "residual_rms": 0.0}
    ida, idb = getattr(img_a, "image_id", "a"), getattr(img_b, "image_id", "b")
    if result is not None:
        t0 = time.perf_counter()
        placements = [K.Placement(ida, RigidTransform.identity()), K.Placement(idb, result.transform.inverse())]
        pa, pb = _compositor_pixels(img_a), _compositor_pixels(img_b)
        canvas = K.compute_canvas(placements, {ida: tuple(pa.shape[:2]), idb: tuple(pb.shape[:2])})
        composite = K.warp_and_blend({ida: pa, idb: pb}, placements, canvas, blend=cfg.blend, resample=cfg.resample)
        stitch_s += time.perf_counter() - t0
        registration.update(theta_deg=math.degrees(result.transform.theta), t_x=result.transform.t_x,
                            t_y=result.transform.t_y, inliers=len(result.inliers), residual_rms=result.residual_rms)
    report = {
        "success": result is not None, "image_a": ida, "image_b": idb,
        "features": {ida: prep_a.feature_count, idb: prep_b.feature_count},
        "matched_pairs": len(pairs), "registration": registration,
        "stage_seconds": {"detection": prep_a.detect_seconds + prep_b.detect_seconds,
                          "description": prep_a.describe_seconds + prep_b.describe_seconds,
                          "matching": match_s, "stitching": stitch_s},
        "total_seconds": time.perf_counter() - start,
    }
    return StitchResult(result is not None, result.transform if result else None, result, composite, report)


@functools.lru_cache(maxsize=65536)
def pair_seed(seed: int, a: int, b: int) -> int:
    """mosaic.py:75-76 (SeedSequence hashing costs ~10 us: cached, it is a pure function)."""
    return int(np.random.SeedSequence([seed, a, b]).generate_state(1)[0])



@dataclass(eq=False)
class HostFeatures:
    """Host (pinned) result of ``prepare_batch_host``."""

    row: torch.Tensor  # int32 [B, cap]
    col: torch.Tensor
    value: torch.Tensor  # float64 [B, cap]
    count: torch.Tensor  # int32 [B]
    descriptors: torch.Tensor  # float32 [B, cap, D]


def alloc_plan_cap(nr: int, nc: int, cfg: PipelineConfig) -> int:
    """Per-image keypoint capacity of the detect plan (count law upper bound)."""
    import ctypes as C

    from . import _lib

    sizes = cfg.scale_set().sizes
    cap, ws = C.c_int64(), C.c_size_t()
    _lib.check(_lib.lib().ps_detect_plan(1, nr, nc, _lib.int32_array(sizes), len(sizes), 1, C.byref(cap),
                                         C.byref(ws)), "detect")
    return cap.value


def alloc_host_features(batch: int, nr: int, nc: int, cfg: PipelineConfig) -> HostFeatures:
    """Pinned output buffers for ``prepare_batch_host`` (allocate once, reuse)."""
    K, D = alloc_plan_cap(nr, nc, cfg), cfg.d * cfg.d * 8
    pin = dict(pin_memory=True)
    return HostFeatures(torch.empty((batch, K), dtype=torch.int32, **pin),
                        torch.empty((batch, K), dtype=torch.int32, **pin),
                        torch.empty((batch, K), dtype=torch.float64, **pin),
                        torch.empty((batch,), dtype=torch.int32, **pin),
                        torch.empty((batch, K, D), dtype=torch.float32, **pin))


class BatchPreparer:
    """Host-to-host detect + describe of many same-sized 8-bit images (grey
    [B, nr, nc], or RGB [B, nr, nc, 3] with ``rgb=True``: BT.601 grey on the
    device).

    Chunks of ``chunk`` images flow through a 3-deep stream pipeline: the
    host->device copy of chunk i+1 and the device->host copy of chunk i-1
    overlap the kernels of chunk i.  Device buffers are allocated once.
    """

    def __init__(self, nr: int, nc: int, cfg: PipelineConfig, chunk: int = 8, depth: int = 3, device_id=None,
                 rgb: bool = False):
        self.cfg, self.nr, self.nc, self.chunk, self.depth = cfg, nr, nc, chunk, depth
        self.alpha = cfg.alpha if cfg.alpha is not None else default_alpha(nr, nc)
        self.sizes = cfg.scale_set().sizes
        self.dcfg = cfg.descriptor_config()
        dev = torch.device("cuda", torch.cuda.current_device() if device_id is None else device_id)
        self.streams = [torch.cuda.Stream(dev) for _ in range(depth)]
        shape = (chunk, nr, nc, 3) if rgb else (chunk, nr, nc)
        self.img = [torch.empty(shape, dtype=torch.uint8, device=dev) for _ in range(depth)]
        self.kind, self.lut = "u8", None
        if rgb:
            from .ingest import gray_source

            self.kind, self.lut = "rgb8", gray_source(dev)
        K = alloc_plan_cap(nr, nc, cfg)
        D = cfg.d * cfg.d * 8
        self.desc = [torch.empty((chunk, K, D), dtype=torch.float32, device=dev) for _ in range(depth)]
        self.out = [None] * depth
        self.dev = dev

    def run(self, host_images: torch.Tensor, out: HostFeatures) -> HostFeatures:
        B = host_images.shape[0]
        done = [None] * self.depth
        for i, b0 in enumerate(range(0, B, self.chunk)):
            slot = i % self.depth
            s = self.streams[slot]
            b1 = min(B, b0 + self.chunk)
            n = b1 - b0
            if done[slot] is not None:
                done[slot].synchronize()  # slot's previous D2H finished -> buffers reusable
            with torch.cuda.stream(s):
                self.img[slot][:n].copy_(host_images[b0:b1], non_blocking=True)
                dimg = device.DeviceImages(self.img[slot][:n], self.kind, self.alpha, self.lut)
                kp = device.detect(dimg, self.sizes, dedupe=True, meta=False, stream=s)
                d32 = self.desc[slot][:n]
                device.describe_into(dimg, kp, self.dcfg, d32, scale_set=kp.scale_set, stream=s)
                out.row[b0:b1].copy_(kp.row, non_blocking=True)
                out.col[b0:b1].copy_(kp.col, non_blocking=True)
                out.value[b0:b1].copy_(kp.value, non_blocking=True)
                out.count[b0:b1].copy_(kp.count, non_blocking=True)
                out.descriptors[b0:b1].copy_(d32, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s)
                done[slot] = ev
                self.out[slot] = (kp, d32)  # keep device buffers alive until the copies finish
        for ev in done:
            if ev is not None:
                ev.synchronize()
        return out


def prepare_batch_host(host_images, cfg: PipelineConfig, out: HostFeatures | None = None, chunk: int = 8):
    """Host 8-bit images [B, nr, nc] (or RGB [B, nr, nc, 3]) -> host keypoints
    + float32 descriptors."""
    t = host_images if isinstance(host_images, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(host_images))
    rgb = t.dim() == 4
    B, nr, nc = t.shape[:3]
    if out is None:
        out = alloc_host_features(B, nr, nc, cfg)
    return BatchPreparer(nr, nc, cfg, chunk=chunk, rgb=rgb).run(t, out)
