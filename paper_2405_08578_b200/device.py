"""Tensor-in / tensor-out API of the B200 hot path (torch CUDA tensors).

Every function here is a thin call into the C-ABI library (``_lib``); torch
is only used for device memory, streams and small host<->device copies.
There is no CPU path: on a machine without CUDA these functions raise.
"""

from __future__ import annotations

import ctypes as C
import functools
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, RegistrationError
from .records import default_alpha


def _require_cuda(t: torch.Tensor, what: str) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (peakstitch_b200 has no CPU path)")


def _stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


# ---------------------------------------------------------------------------
# images
# ---------------------------------------------------------------------------

@dataclass
class DeviceImages:
    """A batch of same-sized rasters on the GPU.

    kind "u8"     : raw 8-bit intensities, ramp fused with ``alpha``;
    kind "f64raw" : float64 intensities, ramp fused with ``alpha``;
    kind "f64"    : already-ramped float64 raster (alpha informational);
    kind "rgb8"   : interleaved 8-bit RGB [B, nr, nc, 3]; grey from the run
                    host's BT.601 table (``ingest.gray_lut``), ramp fused.
    """

    data: torch.Tensor  # [B, nr, nc] (rgb8: [B, nr, nc, 3])
    kind: str
    alpha: float
    lut: torch.Tensor | None = None

    @property
    def batch(self) -> int:
        return int(self.data.shape[0])

    @property
    def nr(self) -> int:
        return int(self.data.shape[1])

    @property
    def nc(self) -> int:
        return int(self.data.shape[2])

    def c_struct(self) -> _lib.ImageBatch:
        d = self.data
        if self.kind == "rgb8":
            if d.dim() != 4 or d.shape[3] != 3 or d.stride(3) != 1 or d.stride(2) != 3 or d.stride(1) % 3 \
                    or d.stride(0) % 3:
                raise ValueError("RGB images must be [B, nr, nc, 3] with interleaved channels")
            return _lib.ImageBatch(d.data_ptr(), _lib.PS_PIXELS_RGB8, d.shape[0], d.shape[1], d.shape[2],
                                   d.stride(1) // 3, (d.stride(0) if d.shape[0] > 1 else d.stride(1) * d.shape[1]) // 3,
                                   float(self.alpha), self.lut.data_ptr() if self.lut is not None else None)
        if d.dim() != 3 or d.stride(2) != 1:
            raise ValueError("images must be [B, nr, nc] with unit column stride")
        ptype = {"u8": _lib.PS_PIXELS_U8, "f64": _lib.PS_PIXELS_F64, "f64raw": _lib.PS_PIXELS_F64_RAW}[self.kind]
        return _lib.ImageBatch(d.data_ptr(), ptype, d.shape[0], d.shape[1], d.shape[2], d.stride(1),
                               d.stride(0) if d.shape[0] > 1 else d.stride(1) * d.shape[1], float(self.alpha), None)


def as_device_images(images, alpha=None, *, ramped=False, rgb=False, device=None) -> DeviceImages:
    """Wrap a [B, nr, nc] / [nr, nc] uint8 or float64 tensor (uploads if on
    CPU); with ``rgb=True`` (or a 4-D tensor) a [B, nr, nc, 3] / [nr, nc, 3]
    uint8 RGB batch whose grey is the reference's BT.601 (imaging.py:66-68)."""
    if isinstance(images, DeviceImages):
        return images
    t = images if isinstance(images, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(images))
    if rgb or t.dim() == 4:
        from .ingest import gray_source

        if t.dim() == 3:
            t = t.unsqueeze(0)
        if t.dim() != 4 or t.shape[3] != 3 or t.dtype != torch.uint8:
            raise ValueError("RGB input must be uint8 [B, nr, nc, 3] or [nr, nc, 3]")
        if not t.is_cuda:
            t = t.to(device or "cuda", non_blocking=False)
        t = t.contiguous()
        if alpha is None:
            alpha = default_alpha(t.shape[1], t.shape[2])
        return DeviceImages(t, "rgb8", float(alpha), gray_source(t.device))
    if t.dim() == 2:
        t = t.unsqueeze(0)
    if not t.is_cuda:
        t = t.to(device or "cuda", non_blocking=False)
    if t.dtype == torch.uint8:
        kind = "u8"
    elif t.dtype == torch.float64:
        kind = "f64" if ramped else "f64raw"
    else:
        t, kind = t.to(torch.float64), ("f64" if ramped else "f64raw")
    if t.stride(2) != 1:
        t = t.contiguous()
    if alpha is None:
        alpha = default_alpha(t.shape[1], t.shape[2])
    return DeviceImages(t, kind, float(alpha))


# ---------------------------------------------------------------------------
# keypoints
# ---------------------------------------------------------------------------

@dataclass
class Keypoints:
    """Per-image keypoint slots [B, cap]; image b's valid slots are [0, count[b])."""

    row: torch.Tensor
    col: torch.Tensor
    value: torch.Tensor
    count: torch.Tensor
    scale: torch.Tensor | None = None
    polarity: torch.Tensor | None = None
    window: torch.Tensor | None = None
    default_scale: int = 0
    scale_set: tuple = ()
    # window side L when slot 2w / 2w+1 is the max / min of window w of L's
    # row-major grid (ps_detect with dedupe and one evaluated scale), else 0
    window_slots: int = 0

    @property
    def cap(self) -> int:
        return int(self.row.shape[1])

    @property
    def batch(self) -> int:
        return int(self.row.shape[0])

    def c_struct(self) -> _lib.KeypointsC:
        def p(t):
            return None if t is None else t.data_ptr()

        return _lib.KeypointsC(p(self.row), p(self.col), p(self.value), p(self.scale), p(self.polarity),
                               p(self.window), p(self.count), self.cap)

    def image(self, b: int) -> dict:
        """Host copy of image b's keypoints (numpy arrays)."""
        n = int(self.count[b].item())
        out = dict(row=self.row[b, :n].cpu().numpy(), col=self.col[b, :n].cpu().numpy(),
                   value=self.value[b, :n].cpu().numpy())
        for k in ("scale", "polarity", "window"):
            t = getattr(self, k)
            if t is not None:
                out[k] = t[b, :n].cpu().numpy()
        return out


def _window_slots(sizes, dedupe) -> int:
    """L_min when ps_detect evaluates only L_min (with dedupe, a scale that is
    a multiple of a smaller one contributes only duplicates, csrc/detect.cu):
    its output is then window w's max / min in slots 2w / 2w+1."""
    s = sorted(sizes)
    evaluated = [x for i, x in enumerate(s) if not any(x % y == 0 for y in s[:i])]
    return s[0] if dedupe and evaluated == [s[0]] else 0


def _describe_policy(policy: str, kp: "Keypoints") -> int:
    flag = _lib.PS_DESCRIBE_WINDOW_SLOTS if (kp.window_slots and kp.window_slots == kp.default_scale) else 0
    return DESCRIBE_POLICIES[policy] | flag


def detect(images, scales, *, alpha=None, dedupe=True, ramped=False, meta=True, stream=None) -> Keypoints:
    """Multiscale window extrema of every image (detector.py:154-172).

    ``meta=False`` skips writing scale/polarity/window (they are implied by
    the slot for single-evaluated-scale plans: slot 2w -> window w max,
    2w+1 -> min, scale = scales[0]).
    """
    im = as_device_images(images, alpha, ramped=ramped)
    sizes = [int(s) for s in (scales.sizes if hasattr(scales, "sizes") else scales)]
    L = _lib.lib()
    arr = _lib.int32_array(sizes)
    cap, wsb = C.c_int64(), C.c_size_t()
    _lib.check(L.ps_detect_plan(im.batch, im.nr, im.nc, arr, len(sizes), int(bool(dedupe)), C.byref(cap),
                                C.byref(wsb)), "detect")
    dev = im.data.device
    B, K = im.batch, cap.value
    kp = Keypoints(
        row=torch.empty((B, K), dtype=torch.int32, device=dev),
        col=torch.empty((B, K), dtype=torch.int32, device=dev),
        value=torch.empty((B, K), dtype=torch.float64, device=dev),
        count=torch.empty((B,), dtype=torch.int32, device=dev),
        scale=torch.empty((B, K), dtype=torch.int32, device=dev) if meta else None,
        polarity=torch.empty((B, K), dtype=torch.int8, device=dev) if meta else None,
        window=torch.empty((B, K), dtype=torch.int32, device=dev) if meta else None,
        default_scale=sizes[0],
        scale_set=tuple(sizes),
        window_slots=_window_slots(sizes, dedupe),
    )
    ws = _workspace(wsb.value, dev)
    ib, kc = im.c_struct(), kp.c_struct()
    _lib.check(L.ps_detect(C.byref(ib), arr, len(sizes), int(bool(dedupe)), C.byref(kc), C.c_void_p(ws.data_ptr()),
                           wsb.value, C.c_void_p(_stream_ptr(stream))), "detect")
    kp._ws = ws  # keep the workspace alive until the stream has consumed it
    return kp


DESCRIBE_POLICIES = {"auto": _lib.PS_DESCRIBE_AUTO, "general": _lib.PS_DESCRIBE_GENERAL,
                     "single": _lib.PS_DESCRIBE_SINGLE, "precise": _lib.PS_DESCRIBE_PRECISE}


def describe(images, kp: Keypoints, cfg, *, alpha=None, ramped=False, scale_set=None, out64=False,
             out32=True, stream=None, policy: str = "auto"):
    """Descriptors of every keypoint slot (descriptor.py:219-269).

    Returns float32 [B, cap, D] (and float64 if ``out64``); slots >= count
    are left unwritten (zero-initialised here).
    """
    im = as_device_images(images, alpha, ramped=ramped)
    D = cfg.d * cfg.d * 8
    if scale_set is None:
        scale_set = kp.scale_set or (kp.default_scale,)
    sset = [int(s) for s in (scale_set.sizes if hasattr(scale_set, "sizes") else scale_set)]
    dev = im.data.device
    d32 = torch.zeros((kp.batch, kp.cap, D), dtype=torch.float32, device=dev) if out32 else None
    d64 = torch.zeros((kp.batch, kp.cap, D), dtype=torch.float64, device=dev) if out64 else None
    L = _lib.lib()
    ib, kc = im.c_struct(), kp.c_struct()
    _lib.check(L.ps_describe_ex(C.byref(ib), C.byref(kc), int(kp.default_scale), _lib.int32_array(sset), len(sset),
                                float(cfg.beta0), int(cfg.d), int(cfg.l_max), int(bool(cfg.orientation_normalize)),
                                _ptr(d32), _ptr(d64), _describe_policy(policy, kp), C.c_void_p(_stream_ptr(stream))),
               "describe")
    if out64 and out32:
        return d32, d64
    return d64 if out64 else d32


def describe_into(images, kp: Keypoints, cfg, out32: torch.Tensor, *, scale_set=None, stream=None,
                  policy: str = "auto") -> None:
    """As ``describe`` into a preallocated float32 [B, cap, D] buffer (no allocation)."""
    im = images if isinstance(images, DeviceImages) else as_device_images(images)
    sset = [int(s) for s in (scale_set or kp.scale_set or (kp.default_scale,))]
    ib, kc = im.c_struct(), kp.c_struct()
    _lib.check(_lib.lib().ps_describe_ex(C.byref(ib), C.byref(kc), int(kp.default_scale), _lib.int32_array(sset),
                                         len(sset), float(cfg.beta0), int(cfg.d), int(cfg.l_max),
                                         int(bool(cfg.orientation_normalize)), _ptr(out32), None,
                                         _describe_policy(policy, kp), C.c_void_p(_stream_ptr(stream))), "describe")


# ---------------------------------------------------------------------------
# matching
# ---------------------------------------------------------------------------

STRATEGIES = {"nearest_neighbor": _lib.PS_MATCH_NEAREST, "threshold_all": _lib.PS_MATCH_THRESHOLD_ALL,
              "ratio_test": _lib.PS_MATCH_RATIO}
# explicit per-call kernel path (include/peakstitch_b200.h PS_MATCH_FORCE_*); results are identical
PATHS = {"auto": 0, "exact": _lib.PS_MATCH_FORCE_EXACT, "tensor": _lib.PS_MATCH_FORCE_TC}


def _path_flag(path: str) -> int:
    if path not in PATHS:
        raise ValueError(f"unknown match path {path!r} (auto / exact / tensor)")
    return PATHS[path]


def match(desc1: torch.Tensor, desc2: torch.Tensor, delta_s: float = 0.35, strategy: str = "nearest_neighbor",
          cap: int | None = None, stream=None, path: str = "auto"):
    """Matches sorted by (delta, ref1, ref2) (matcher.py:57-95).

    ``strategy`` "ratio_test" is the extra Lowe-ratio strategy (not in the
    reference): ``delta_s`` is then the ratio r in (0, 1] and row i keeps its
    first nearest neighbour when d1 < r * d2.
    Returns device tensors (ref1 int32 [M], ref2 int32 [M], delta float64 [M]).
    """
    if strategy not in STRATEGIES:
        raise ConfigError(f"unknown match strategy {strategy!r}")
    if delta_s <= 0:
        raise ConfigError(f"delta_s must be positive, got {delta_s}")
    # float64 inputs are matched exactly as given; anything else as float32
    dt = torch.float64 if (desc1.dtype == torch.float64 or desc2.dtype == torch.float64) else torch.float32
    d1 = desc1.to(dt).contiguous()
    d2 = desc2.to(dt).contiguous()
    _require_cuda(d1, "desc1")
    n1, n2 = int(d1.shape[0]), int(d2.shape[0])
    dim = int(d1.shape[1]) if d1.dim() == 2 else 128
    dev = d1.device
    if n1 == 0 or n2 == 0:
        e = torch.zeros(0, dtype=torch.int32, device=dev)
        return e, e.clone(), torch.zeros(0, dtype=torch.float64, device=dev)
    strat = STRATEGIES[strategy]
    if cap is None:
        cap = {_lib.PS_MATCH_NEAREST: min(n1, n2), _lib.PS_MATCH_RATIO: n1}.get(strat, max(4 * (n1 + n2), 1024))
    strat |= _path_flag(path)
    L = _lib.lib()
    while True:
        wsb = C.c_size_t()
        _lib.check(L.ps_match_plan(n1, n2, dim, strat, cap, C.byref(wsb)), "match")
        ws = _workspace(wsb.value, dev)
        r1 = torch.empty(cap, dtype=torch.int32, device=dev)
        r2 = torch.empty(cap, dtype=torch.int32, device=dev)
        dl = torch.empty(cap, dtype=torch.float64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.check(L.ps_match(_ptr(d1), n1, _ptr(d2), n2, dim, int(dt == torch.float64), float(delta_s), strat, _ptr(r1), _ptr(r2), _ptr(dl),
                              _ptr(cnt), cap, _ptr(ws), wsb.value, C.c_void_p(_stream_ptr(stream))), "match")
        m = int(cnt.item())
        if m <= cap:
            return r1[:m], r2[:m], dl[:m]
        cap = m  # threshold_all overflow: retry with the exact size


def match_async(desc1: torch.Tensor, desc2: torch.Tensor, delta_s: float = 0.35, *, out_count=None, stream=None,
                path: str = "auto"):
    """nearest_neighbor matching enqueued with no host synchronisation
    (ps_match_async; same results as ``match``).  Returns device tensors
    (ref1 int32 [cap], ref2 int32 [cap], delta float64 [cap], count int64 [1]);
    rows [0, count) are valid, sorted by (delta, ref1, ref2).  ``out_count``
    may be a caller-provided int64 [1] view (e.g. one slot of a batch)."""
    if delta_s <= 0:
        raise ConfigError(f"delta_s must be positive, got {delta_s}")
    dt = torch.float64 if (desc1.dtype == torch.float64 or desc2.dtype == torch.float64) else torch.float32
    d1, d2 = desc1.to(dt).contiguous(), desc2.to(dt).contiguous()
    _require_cuda(d1, "desc1")
    n1, n2 = int(d1.shape[0]), int(d2.shape[0])
    dim = int(d1.shape[1]) if d1.dim() == 2 else 128
    dev = d1.device
    cap = max(min(n1, n2), 1)
    cnt = out_count if out_count is not None else torch.zeros(1, dtype=torch.int64, device=dev)
    r1 = torch.empty(cap, dtype=torch.int32, device=dev)
    r2 = torch.empty(cap, dtype=torch.int32, device=dev)
    dl = torch.empty(cap, dtype=torch.float64, device=dev)
    if n1 == 0 or n2 == 0:
        cnt.zero_()
        return r1, r2, dl, cnt
    L = _lib.lib()
    wsb = C.c_size_t()
    strat = _lib.PS_MATCH_NEAREST | _path_flag(path)
    _lib.check(L.ps_match_plan(n1, n2, dim, strat, cap, C.byref(wsb)), "match")
    ws = _workspace(wsb.value, dev)
    _lib.check(L.ps_match_async(_ptr(d1), n1, _ptr(d2), n2, dim, int(dt == torch.float64), float(delta_s),
                                strat, _ptr(r1), _ptr(r2), _ptr(dl), _ptr(cnt), cap, _ptr(ws),
                                wsb.value, C.c_void_p(_stream_ptr(stream))), "match")
    return r1, r2, dl, cnt


def match_many_async(pairs, delta_s: float, counts: torch.Tensor, *, streams=None) -> list:
    """Enqueue nearest_neighbor matching of every pair with no host
    synchronisation (capturable in a CUDA graph): pair q's count goes to
    counts[q] (device int64).  Returns [(ref1, ref2, delta), ...] full-capacity
    device buffers, valid rows [0, counts[q])."""
    if not pairs:
        return []
    dev = pairs[0][0].device
    cur = torch.cuda.current_stream(dev)
    outs = []
    if streams:
        ready = cur.record_event()
        for s in streams:
            s.wait_event(ready)
    for q, (a, b) in enumerate(pairs):
        s = streams[q % len(streams)] if streams else None
        if s is not None:
            with torch.cuda.stream(s):
                o = match_async(a, b, delta_s, out_count=counts[q:q + 1], stream=s)
                for t in (a, b) + o[:3]:
                    t.record_stream(s)
        else:
            o = match_async(a, b, delta_s, out_count=counts[q:q + 1])
        outs.append(o[:3])
    if streams:
        for s in streams:
            cur.wait_stream(s)
    return outs


def match_many(pairs, delta_s: float = 0.35, *, streams=None):
    """nearest_neighbor matching of many descriptor-set pairs with ONE host
    synchronisation: every pair is enqueued asynchronously (round-robin over
    ``streams`` when given, each joined back to the current stream), then all
    match counts are read with one copy.  ``pairs`` = [(desc1, desc2), ...];
    returns [(ref1, ref2, delta), ...] device tensors trimmed to their counts."""
    if not pairs:
        return []
    counts = torch.zeros(len(pairs), dtype=torch.int64, device=pairs[0][0].device)
    outs = match_many_async(pairs, delta_s, counts, streams=streams)
    m = counts.cpu().tolist()
    return [(r1[:k], r2[:k], dl[:k]) for (r1, r2, dl), k in zip(outs, m)]


BATCH_MAX_SETS, BATCH_MAX_PAIRS = 512, 256  # ps_match_batch_async limits per call


def match_batch_async(sets, pairs, delta_s: float = 0.35, *, out_count=None, stream=None, set_counts=None):
    """nearest_neighbor matching of many pairs over shared descriptor sets as
    one launch sequence (ps_match_batch_async): each set's duplicate grouping
    and tensor-core operand tiles are built once however many pairs use it,
    and every stage is one launch for all pairs.  No host synchronisation
    (capturable).  ``sets`` = [desc [n_s, 128] device tensors], ``pairs`` =
    [(a, b), ...] set indices.  Returns (ref1 int32 [P, S], ref2 int32 [P, S],
    delta float64 [P, S], count int64 [P]) with S = max over pairs of
    min(n_a, n_b); row q holds pair q's matches in [0, count[q]), sorted by
    (delta, ref1, ref2) -- the same as ``match`` pair by pair.

    ``set_counts`` (optional): one device int32 tensor (1 element) or None
    per set, the set's live row count; the set tensor is then its capacity and
    the kernels read the count on the device, so a graph captured over this
    call stays valid when the counts change between replays."""
    if delta_s <= 0:
        raise ConfigError(f"delta_s must be positive, got {delta_s}")
    P = len(pairs)
    if not sets:
        raise ValueError("match_batch_async needs at least one descriptor set")
    dt = torch.float64 if any(s.dtype == torch.float64 for s in sets) else torch.float32
    ds = [s.to(dt).contiguous() for s in sets]
    for d in ds:
        _require_cuda(d, "descriptor set")
        if d.dim() != 2 or int(d.shape[1]) != 128:
            raise ValueError(f"match_batch_async needs [n, 128] descriptor sets, got {tuple(d.shape)}")
    dev = ds[0].device
    rows = [int(d.shape[0]) for d in ds]
    stride = max([min(rows[a], rows[b]) for a, b in pairs] + [1])
    cnt = out_count if out_count is not None else torch.zeros(P, dtype=torch.int64, device=dev)
    r1 = torch.empty((P, stride), dtype=torch.int32, device=dev)
    r2 = torch.empty((P, stride), dtype=torch.int32, device=dev)
    dl = torch.empty((P, stride), dtype=torch.float64, device=dev)
    L = _lib.lib()
    for q0 in range(0, P, BATCH_MAX_PAIRS):
        chunk = list(pairs[q0:q0 + BATCH_MAX_PAIRS])
        used = sorted({s for pr in chunk for s in pr})  # <= 2 x BATCH_MAX_PAIRS = BATCH_MAX_SETS
        local = {s: i for i, s in enumerate(used)}
        S = len(used)
        ptrs = (C.c_void_p * S)(*[ds[s].data_ptr() for s in used])
        cnts = None
        if set_counts is not None:
            for s in used:
                c = set_counts[s]
                if c is not None and (c.dtype != torch.int32 or c.device != dev or c.numel() < 1):
                    raise ValueError("set_counts entries must be device int32 tensors on the sets' device")
            cnts = (C.c_void_p * S)(*[set_counts[s].data_ptr() if set_counts[s] is not None else None
                                      for s in used])
        rows_c = (C.c_int64 * S)(*[rows[s] for s in used])
        pa = (C.c_int32 * len(chunk))(*[local[a] for a, _ in chunk])
        pb = (C.c_int32 * len(chunk))(*[local[b] for _, b in chunk])
        wsb = C.c_size_t()
        _lib.check(L.ps_match_batch_plan(S, rows_c, len(chunk), 128, C.byref(wsb)), "match_batch")
        ws = _workspace(wsb.value, dev)
        _lib.check(L.ps_match_batch_async(S, ptrs, rows_c, cnts, len(chunk), pa, pb, 128, int(dt == torch.float64),
                                          float(delta_s), _ptr(r1[q0:]), _ptr(r2[q0:]), _ptr(dl[q0:]), stride,
                                          _ptr(cnt[q0:]), _ptr(ws), wsb.value, C.c_void_p(_stream_ptr(stream))),
                   "match_batch")
    return r1, r2, dl, cnt


def pair_points(r1, r2, kp1_row, kp1_col, kp2_row, kp2_col, stream=None):
    """(x, y) = (col, row) float64 coordinates of matched pairs (registration.py:143-146)."""
    n = int(r1.shape[0])
    dev = r1.device
    src = torch.empty((n, 2), dtype=torch.float64, device=dev)
    dst = torch.empty((n, 2), dtype=torch.float64, device=dev)
    if n:
        cnt = torch.full((1,), n, dtype=torch.int64, device=dev)  # fill kernel: no host sync
        _lib.check(_lib.lib().ps_pair_points(_ptr(r1), _ptr(r2), _ptr(cnt), _ptr(kp1_row), _ptr(kp1_col),
                                             _ptr(kp2_row), _ptr(kp2_col), _ptr(src), _ptr(dst), n,
                                             C.c_void_p(_stream_ptr(stream))), "pair_points")
    return src, dst


def pair_points_dev(r1, r2, count: torch.Tensor, kp1_row, kp1_col, kp2_row, kp2_col, stream=None):
    """``pair_points`` for full-capacity match buffers whose count is on the
    device (int64 [1]); rows >= count are left unwritten."""
    n = int(r1.shape[0])
    dev = r1.device
    src = torch.empty((n, 2), dtype=torch.float64, device=dev)
    dst = torch.empty((n, 2), dtype=torch.float64, device=dev)
    if n:
        _lib.check(_lib.lib().ps_pair_points(_ptr(r1), _ptr(r2), _ptr(count), _ptr(kp1_row), _ptr(kp1_col),
                                             _ptr(kp2_row), _ptr(kp2_col), _ptr(src), _ptr(dst), n,
                                             C.c_void_p(_stream_ptr(stream))), "pair_points")
    return src, dst


# ---------------------------------------------------------------------------
# registration
# ---------------------------------------------------------------------------

def sample_stream(seed: int, n: int, iterations: int) -> np.ndarray:
    """The reference's RANSAC index stream (registration.py:164, 170-173).

    numpy's PCG64 ``Generator`` is the reference's own RNG; one vector draw
    with highs [n, n-1, n, n-1, ...] equals its alternating scalar calls.
    Host-side by design (seeded sampling is part of the interface).
    """
    rng = np.random.default_rng(seed)
    highs = np.tile(np.array([n, n - 1], dtype=np.int64), iterations)
    v = rng.integers(0, highs).reshape(iterations, 2)
    v[:, 1] += v[:, 1] >= v[:, 0]
    return v.astype(np.int32)


@functools.lru_cache(maxsize=256)
def _pcg_state(seed: int) -> tuple:
    """(state, inc, has_uint32, uinteger) of default_rng(seed) -- SeedSequence
    hashing is the host-side cost of a RANSAC call, so it is cached per seed."""
    st = np.random.default_rng(seed).bit_generator.state
    return int(st["state"]["state"]), int(st["state"]["inc"]), int(st["has_uint32"]), int(st["uinteger"])


def sample_stream_device(seed: int, n: int, iterations: int, device=None, stream=None) -> torch.Tensor:
    """The same stream generated on the GPU (ps_ransac_samples): only the
    seeded PCG64 state comes from numpy (SeedSequence seeding on the host),
    the draws -- jump-ahead per iteration, Lemire bounds, exact sequential
    replay when a rejection occurs -- run on the device.  int32 [iters, 2]."""
    s, inc, has_u32, u32 = _pcg_state(int(seed))
    m64 = (1 << 64) - 1
    out = torch.empty(2 * iterations + 1, dtype=torch.int32, device=device or "cuda")
    _lib.check(_lib.lib().ps_ransac_samples(s >> 64, s & m64, inc >> 64, inc & m64, has_u32,
                                            u32, int(n), int(iterations), _ptr(out),
                                            C.c_void_p(out.data_ptr() + 8 * iterations),
                                            C.c_void_p(_stream_ptr(stream))), "ransac_samples")
    return out[: 2 * iterations].view(iterations, 2)


@dataclass
class RansacOutcome:
    ok: bool
    status: int
    theta: float
    t_x: float
    t_y: float
    inliers: np.ndarray
    consensus: int
    rms: float
    best_iteration: int


def ransac(src: torch.Tensor, dst: torch.Tensor, iterations=2000, inlier_tol=3.0, min_inliers=8, seed=0,
           stream=None) -> RansacOutcome:
    """2-point rigid RANSAC on device (registration.py:149-203)."""
    if iterations < 1 or inlier_tol <= 0 or min_inliers < 2:
        raise ConfigError("invalid RANSAC parameters")
    n = int(src.shape[0])
    if n < min_inliers:
        raise RegistrationError(f"only {n} candidate pairs, need at least {min_inliers}")
    _require_cuda(src, "src")
    dev = src.device
    src = src.to(torch.float64).contiguous()
    dst = dst.to(torch.float64).contiguous()
    samples = sample_stream_device(seed, n, iterations, dev, stream)
    L = _lib.lib()
    wsb = C.c_size_t()
    _lib.check(L.ps_ransac_plan(n, iterations, C.byref(wsb)), "ransac")
    ws = _workspace(wsb.value, dev)
    # one result block: model[3] | rms | info[4] (int64 bits) | mask[n] -- a single device-to-host read
    out = torch.empty(8 + (n + 7) // 8, dtype=torch.float64, device=dev)
    ob = out.view(torch.uint8)
    model, rms, info, mask = out[0:3], out[3:4], out[4:8].view(torch.int64), ob[64:64 + n]
    _lib.check(L.ps_ransac_rigid(_ptr(src), _ptr(dst), n, _ptr(samples), iterations, float(inlier_tol),
                                 int(min_inliers), _ptr(model), _ptr(mask), _ptr(info), _ptr(rms), _ptr(ws),
                                 wsb.value, C.c_void_p(_stream_ptr(stream))), "ransac")
    h = out.cpu()
    model_h, rms_h = h[0:3].numpy(), float(h[3])
    info_h = h[4:8].view(torch.int64).numpy()
    inl = np.flatnonzero(h.view(torch.uint8)[64:64 + n].numpy()).astype(np.int64)
    st = int(info_h[0])
    return RansacOutcome(ok=st == _lib.PS_OK, status=st, theta=float(model_h[0]), t_x=float(model_h[1]),
                         t_y=float(model_h[2]), inliers=inl, consensus=int(info_h[1]), rms=rms_h,
                         best_iteration=int(info_h[3]))


def ransac_async(src: torch.Tensor, dst: torch.Tensor, iterations=2000, inlier_tol=3.0, min_inliers=8, seed=0,
                 *, out=None, stream=None) -> torch.Tensor:
    """``ransac`` enqueued without reading the result back: returns the
    device result block (float64 [8 + ceil(n/8)]: model[3] | rms | info[4] as
    int64 bits | inlier mask bytes) for ``ransac_result``.  ``out`` may be a
    caller-provided block (e.g. one row of a batch)."""
    if iterations < 1 or inlier_tol <= 0 or min_inliers < 2:
        raise ConfigError("invalid RANSAC parameters")
    n = int(src.shape[0])
    if n < min_inliers:
        raise RegistrationError(f"only {n} candidate pairs, need at least {min_inliers}")
    _require_cuda(src, "src")
    dev = src.device
    src = src.to(torch.float64).contiguous()
    dst = dst.to(torch.float64).contiguous()
    samples = sample_stream_device(seed, n, iterations, dev, stream)
    L = _lib.lib()
    wsb = C.c_size_t()
    _lib.check(L.ps_ransac_plan(n, iterations, C.byref(wsb)), "ransac")
    ws = _workspace(wsb.value, dev)
    if out is None:
        out = torch.empty(8 + (n + 7) // 8, dtype=torch.float64, device=dev)
    ob = out.view(torch.uint8)
    model, rms, info, mask = out[0:3], out[3:4], out[4:8].view(torch.int64), ob[64:64 + n]
    _lib.check(L.ps_ransac_rigid(_ptr(src), _ptr(dst), n, _ptr(samples), iterations, float(inlier_tol),
                                 int(min_inliers), _ptr(model), _ptr(mask), _ptr(info), _ptr(rms), _ptr(ws),
                                 wsb.value, C.c_void_p(_stream_ptr(stream))), "ransac")
    return out


def ransac_async_dev(src: torch.Tensor, dst: torch.Tensor, n_dev: torch.Tensor, n_cap: int, iterations: int,
                     inlier_tol: float, min_inliers: int, seed: int, out: torch.Tensor, stream=None) -> None:
    """RANSAC whose correspondence count exists only on the device (n_dev,
    int64 [1], e.g. a match count; src/dst hold >= n_cap rows): the sample
    stream and every kernel read the count there, so a match -> RANSAC chain
    needs no host round trip (ps_ransac_samples_async / ps_ransac_rigid_async).
    Writes the ``ransac_async`` result block layout into ``out`` (length
    >= 8 + ceil(n_cap / 8)); a count below min_inliers reports
    PS_ERR_REGISTRATION in its status word."""
    if iterations < 1 or inlier_tol <= 0 or min_inliers < 2:
        raise ConfigError("invalid RANSAC parameters")
    if n_cap < min_inliers:
        raise RegistrationError(f"only {n_cap} candidate pairs, need at least {min_inliers}")
    dev = src.device
    st, inc, has_u32, u32 = _pcg_state(int(seed))
    m64 = (1 << 64) - 1
    smp = torch.empty(2 * iterations + 1, dtype=torch.int32, device=dev)
    L = _lib.lib()
    sp = C.c_void_p(_stream_ptr(stream))
    _lib.check(L.ps_ransac_samples_async(st >> 64, st & m64, inc >> 64, inc & m64, has_u32, u32, _ptr(n_dev),
                                         int(iterations), _ptr(smp), C.c_void_p(smp.data_ptr() + 8 * iterations),
                                         sp), "ransac_samples")
    wsb = C.c_size_t()
    _lib.check(L.ps_ransac_plan(n_cap, iterations, C.byref(wsb)), "ransac")
    ws = _workspace(wsb.value, dev)
    ob = out.view(torch.uint8)
    _lib.check(L.ps_ransac_rigid_async(_ptr(src), _ptr(dst), _ptr(n_dev), int(n_cap), _ptr(smp), int(iterations),
                                       float(inlier_tol), int(min_inliers), _ptr(out[0:3]),
                                       C.c_void_p(ob.data_ptr() + 64), _ptr(out[4:8]), _ptr(out[3:4]), _ptr(ws),
                                       wsb.value, sp), "ransac")


def register_batch_async(jobs, ref1: torch.Tensor, ref2: torch.Tensor, count: torch.Tensor, iterations: int,
                         inlier_tol: float, min_inliers: int, out: torch.Tensor, stream=None) -> None:
    """Point gather + RANSAC of many matched pairs as one launch per stage
    (ps_register_batch_async; results equal pair_points_dev +
    ransac_async_dev pair by pair).  ``jobs`` = [(row1, col1, row2, col2,
    n_cap, seed) or None (skipped), ...] for the rows of ``ref1`` / ``ref2``
    (int32 [P, S]) and ``count`` (int64 [P]); pair q's ``ransac_async``
    result block goes to ``out[q]`` (float64 [P, >= 8 + ceil(S / 8)])."""
    if iterations < 1 or inlier_tol <= 0 or min_inliers < 2:
        raise ConfigError("invalid RANSAC parameters")
    P, S = int(ref1.shape[0]), int(ref1.shape[1])
    L = _lib.lib()
    m64 = (1 << 64) - 1
    for q0 in range(0, P, BATCH_MAX_PAIRS):
        q1 = min(P, q0 + BATCH_MAX_PAIRS)
        arr = (_lib.RegisterPairC * (q1 - q0))()
        for k, job in enumerate(jobs[q0:q1]):
            if job is None:
                continue
            r1, c1, r2, c2, n_cap, seed = job
            st, inc, has_u32, u32 = _pcg_state(int(seed))
            arr[k] = _lib.RegisterPairC(r1.data_ptr(), c1.data_ptr(), r2.data_ptr(), c2.data_ptr(), int(n_cap),
                                        st >> 64, st & m64, inc >> 64, inc & m64, has_u32, u32, 1)
        wsb = C.c_size_t()
        _lib.check(L.ps_register_batch_plan(q1 - q0, S, int(iterations), C.byref(wsb)), "register_batch")
        ws = _workspace(wsb.value, ref1.device)
        _lib.check(L.ps_register_batch_async(q1 - q0, arr, _ptr(ref1[q0:]), _ptr(ref2[q0:]), S, _ptr(count[q0:]),
                                             int(iterations), float(inlier_tol), int(min_inliers), _ptr(out[q0:]),
                                             int(out.stride(0)), _ptr(ws), wsb.value,
                                             C.c_void_p(_stream_ptr(stream))), "register_batch")


def ransac_result(h: torch.Tensor, n: int) -> RansacOutcome:
    """Decode a host copy of a ``ransac_async`` result block."""
    model_h, rms_h = h[0:3].numpy(), float(h[3])
    info_h = h[4:8].view(torch.int64).numpy()
    inl = np.flatnonzero(h.view(torch.uint8)[64:64 + n].numpy()).astype(np.int64)
    st = int(info_h[0])
    return RansacOutcome(ok=st == _lib.PS_OK, status=st, theta=float(model_h[0]), t_x=float(model_h[1]),
                         t_y=float(model_h[2]), inliers=inl, consensus=int(info_h[1]), rms=rms_h,
                         best_iteration=int(info_h[3]))


def ransac_many(jobs, *, streams=None) -> list:
    """Many RANSAC runs with ONE result read-back.  ``jobs`` = [(src, dst,
    iterations, inlier_tol, min_inliers, seed), ...] (every src with at least
    min_inliers rows); returns [RansacOutcome, ...] in order."""
    if not jobs:
        return []
    dev = jobs[0][0].device
    width = max(8 + (int(j[0].shape[0]) + 7) // 8 for j in jobs)
    block = torch.empty((len(jobs), width), dtype=torch.float64, device=dev)
    cur = torch.cuda.current_stream(dev)
    if streams:
        ready = cur.record_event()
        for s in streams:
            s.wait_event(ready)
    for q, (src, dst, iters, tol, mi, seed) in enumerate(jobs):
        n = int(src.shape[0])
        row = block[q, : 8 + (n + 7) // 8]
        s = streams[q % len(streams)] if streams else None
        if s is not None:
            with torch.cuda.stream(s):
                ransac_async(src, dst, iters, tol, mi, seed, out=row, stream=s)
                src.record_stream(s)
                dst.record_stream(s)
        else:
            ransac_async(src, dst, iters, tol, mi, seed, out=row)
    if streams:
        for s in streams:
            cur.wait_stream(s)
        block.record_stream(cur)
    h = block.cpu()
    return [ransac_result(h[q], int(j[0].shape[0])) for q, j in enumerate(jobs)]


def estimate(src: torch.Tensor, dst: torch.Tensor, stream=None):
    """Least-squares rigid fit (registration.py:107-131) -> (theta, t_x, t_y, status)."""
    _require_cuda(src, "src")
    dev = src.device
    src = src.to(torch.float64).contiguous()
    dst = dst.to(torch.float64).contiguous()
    model = torch.empty(3, dtype=torch.float64, device=dev)
    info = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.check(_lib.lib().ps_estimate_rigid(_ptr(src), _ptr(dst), int(src.shape[0]), _ptr(model), _ptr(info),
                                            C.c_void_p(_stream_ptr(stream))), "estimate_rigid")
    m = model.cpu().numpy()
    return float(m[0]), float(m[1]), float(m[2]), int(info.item())


def kernel_launches() -> int:
    return _lib.kernel_launches()


def nearest(X: torch.Tensor, Y: torch.Tensor, stream=None, path: str = "auto"):
    """Exact first-argmin nearest row of Y for every row of X (one direction of
    nearest_neighbor matching).  Returns (index int32 [nx], dist float64 [nx])."""
    dt = torch.float64 if (X.dtype == torch.float64 or Y.dtype == torch.float64) else torch.float32
    X, Y = X.to(dt).contiguous(), Y.to(dt).contiguous()
    _require_cuda(X, "X")
    nx, ny, dim = int(X.shape[0]), int(Y.shape[0]), int(X.shape[1])
    idx = torch.empty(nx, dtype=torch.int32, device=X.device)
    dist = torch.empty(nx, dtype=torch.float64, device=X.device)
    if nx == 0:
        return idx, dist
    L = _lib.lib()
    wsb = C.c_size_t()
    flags = _path_flag(path)
    _lib.check(L.ps_nearest_plan(nx, ny, dim, flags, C.byref(wsb)), "nearest")
    ws = _workspace(wsb.value, X.device)
    _lib.check(L.ps_nearest(_ptr(X), nx, _ptr(Y), ny, dim, int(dt == torch.float64), flags, _ptr(idx), _ptr(dist), _ptr(ws),
                            wsb.value, C.c_void_p(_stream_ptr(stream))), "nearest")
    return idx, dist


def match_stats() -> dict:
    """Counters of this thread's last tensor-core match (see ps_match_stats)."""
    arr = (C.c_int64 * 8)()
    _lib.lib().ps_match_stats(arr, 8)
    keys = ("distinct_rows_a", "distinct_rows_b", "candidate_columns", "enumerated_rows", "enumerated_pairs",
            "mma_flops", "passes")
    return {k: int(arr[i]) for i, k in enumerate(keys)}
