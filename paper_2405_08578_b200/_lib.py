"""ctypes binding of the C-ABI library ``libpeakstitch_b200.so``.

The library is built in-tree (``__graft_entry__.build()`` / ``make -C
paper_2405_08578_b200/csrc``).  There is no fallback: if the shared object
is missing or does not load, every hot-path entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, DegenerateSampleError, RegistrationError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpeakstitch_b200.so")

PS_OK, PS_ERR_CONFIG, PS_ERR_VALUE, PS_ERR_DEGENERATE, PS_ERR_REGISTRATION = 0, 1, 2, 3, 4
PS_ERR_CUDA, PS_ERR_ARGUMENT, PS_ERR_CAPACITY = 5, 6, 7
PS_PIXELS_U8, PS_PIXELS_F64, PS_PIXELS_F64_RAW, PS_PIXELS_RGB8 = 0, 1, 2, 3
ABI_VERSION = 6
PS_MATCH_NEAREST, PS_MATCH_THRESHOLD_ALL, PS_MATCH_RATIO = 0, 1, 2
PS_MATCH_FORCE_EXACT, PS_MATCH_FORCE_TC = 0x100, 0x200  # per-call path selection (OR-ed into the strategy)
PS_DESCRIBE_AUTO, PS_DESCRIBE_GENERAL, PS_DESCRIBE_SINGLE, PS_DESCRIBE_PRECISE = 0, 1, 2, 3
PS_DESCRIBE_WINDOW_SLOTS = 0x100  # include/peakstitch_b200.h: slots follow the default scale's window grid


class ImageBatch(C.Structure):
    _fields_ = [("data", C.c_void_p), ("pixel_type", C.c_int32), ("batch", C.c_int32),
                ("nr", C.c_int32), ("nc", C.c_int32), ("row_pitch", C.c_int64),
                ("image_stride", C.c_int64), ("alpha", C.c_double), ("gray_lut", C.c_void_p)]


class KeypointsC(C.Structure):
    _fields_ = [("row", C.c_void_p), ("col", C.c_void_p), ("value", C.c_void_p),
                ("scale", C.c_void_p), ("polarity", C.c_void_p), ("window", C.c_void_p),
                ("count", C.c_void_p), ("cap", C.c_int64)]


class PlacementC(C.Structure):
    _fields_ = [("data", C.c_void_p), ("pixel_type", C.c_int32), ("nr", C.c_int32), ("nc", C.c_int32),
                ("r_lo", C.c_int32), ("r_hi", C.c_int32), ("c_lo", C.c_int32), ("c_hi", C.c_int32),
                ("pad_", C.c_int32), ("row_pitch", C.c_int64), ("cos_t", C.c_double), ("sin_t", C.c_double),
                ("t_x", C.c_double), ("t_y", C.c_double)]


class RegisterPairC(C.Structure):
    _fields_ = [("row1", C.c_void_p), ("col1", C.c_void_p), ("row2", C.c_void_p), ("col2", C.c_void_p),
                ("n_cap", C.c_int64), ("state_hi", C.c_uint64), ("state_lo", C.c_uint64),
                ("inc_hi", C.c_uint64), ("inc_lo", C.c_uint64), ("has_uint32", C.c_int32),
                ("uinteger", C.c_uint32), ("live", C.c_int32)]


PS_BLEND_FEATHER, PS_BLEND_OVERWRITE = 0, 1
PS_RESAMPLE_BILINEAR, PS_RESAMPLE_NEAREST = 0, 1

# exported symbol -> (restype, argtypes); mirrors include/peakstitch_b200.h
SIGNATURES = {
    "ps_abi_version": (C.c_int, []),
    "ps_last_error": (C.c_char_p, []),
    "ps_kernel_launches": (C.c_uint64, []),
    "ps_device_sync": (C.c_int, [C.c_void_p]),
    "ps_probe_fp64_fma": (C.c_int, [C.c_int64, C.c_int32, C.c_void_p, C.POINTER(C.c_double), C.c_void_p]),
    "ps_probe_tmem_read": (C.c_int, [C.c_int64, C.c_int32, C.c_void_p, C.POINTER(C.c_double), C.c_void_p]),
    "ps_detect_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                                 C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_size_t)]),
    "ps_detect": (C.c_int, [C.POINTER(ImageBatch), C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                            C.POINTER(KeypointsC), C.c_void_p, C.c_size_t, C.c_void_p]),
    "ps_describe": (C.c_int, [C.POINTER(ImageBatch), C.POINTER(KeypointsC), C.c_int32,
                              C.POINTER(C.c_int32), C.c_int32, C.c_double, C.c_int32, C.c_int32,
                              C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ps_describe_ex": (C.c_int, [C.POINTER(ImageBatch), C.POINTER(KeypointsC), C.c_int32,
                                 C.POINTER(C.c_int32), C.c_int32, C.c_double, C.c_int32, C.c_int32,
                                 C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "ps_match_plan": (C.c_int, [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int64,
                                C.POINTER(C.c_size_t)]),
    "ps_match": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_double,
                           C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                           C.c_void_p, C.c_size_t, C.c_void_p]),
    "ps_match_async": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_double,
                                 C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                 C.c_void_p, C.c_size_t, C.c_void_p]),
    "ps_pair_points": (C.c_int, [C.c_void_p] * 9 + [C.c_int64, C.c_void_p]),
    "ps_register_batch_plan": (C.c_int, [C.c_int32, C.c_int64, C.c_int32, C.POINTER(C.c_size_t)]),
    "ps_register_batch_async": (C.c_int, [C.c_int32, C.POINTER(RegisterPairC), C.c_void_p, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.c_int32, C.c_double, C.c_int32, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.c_size_t, C.c_void_p]),
    "ps_match_batch_plan": (C.c_int, [C.c_int32, C.POINTER(C.c_int64), C.c_int32, C.c_int32,
                                      C.POINTER(C.c_size_t)]),
    "ps_match_batch_async": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_void_p), C.c_int32,
                                       C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                                       C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                       C.c_void_p, C.c_size_t, C.c_void_p]),
    "ps_match_stats": (C.c_int, [C.POINTER(C.c_int64), C.c_int32]),
    "ps_nearest_plan": (C.c_int, [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_size_t)]),
    "ps_nearest": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "ps_ransac_plan": (C.c_int, [C.c_int64, C.c_int32, C.POINTER(C.c_size_t)]),
    "ps_ransac_rigid": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32,
                                  C.c_double, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "ps_ransac_samples": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, C.c_uint32,
                                    C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ps_ransac_rigid_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32,
                                        C.c_double, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "ps_ransac_samples_async": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, C.c_uint32,
                                          C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ps_estimate_rigid": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                    C.c_void_p]),
    "ps_gray_table_check": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "ps_rgb_to_gray": (C.c_int, [C.POINTER(ImageBatch), C.c_void_p, C.c_void_p]),
    "ps_warp_and_blend": (C.c_int, [C.POINTER(PlacementC), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
}

_lib = None


def lib():
    """The loaded library (raises if it is missing: there is no CPU path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not built; run `make -C paper_2405_08578_b200/csrc` "
                "(or __graft_entry__.build()).  peakstitch_b200 has no CPU fallback."
            )
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.ps_abi_version() != ABI_VERSION:
            raise ImportError("libpeakstitch_b200 ABI version mismatch")
        _lib = handle
    return _lib


def last_error() -> str:
    return lib().ps_last_error().decode("utf-8", "replace")


def check(status: int, what: str = "") -> None:
    """Map a ps_status onto the reference's exception taxonomy (errors.py:4-17)."""
    if status == PS_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == PS_ERR_CONFIG:
        raise ConfigError(msg)
    if status == PS_ERR_VALUE:
        raise ValueError(msg)
    if status == PS_ERR_DEGENERATE:
        raise DegenerateSampleError(msg)
    if status == PS_ERR_REGISTRATION:
        raise RegistrationError(msg)
    if status == PS_ERR_ARGUMENT:
        raise ValueError(msg)
    raise RuntimeError(f"peakstitch_b200 CUDA failure ({status}): {msg}")


def kernel_launches() -> int:
    return int(lib().ps_kernel_launches())


def int32_array(values):
    arr = (C.c_int32 * len(values))(*[int(v) for v in values])
    return arr
