"""peakstitch_b200: B200-native (sm_100a) LP-SIFT stitching hot path.

detect -> describe -> match -> RANSAC-score of arXiv 2405.08578 behind the
reference package's own entry points (``detect_features``,
``describe_features``, ``match_features``, ``ransac_rigid``), with CUDA
reached through the C-ABI library ``libpeakstitch_b200.so``
(include/peakstitch_b200.h).  No CPU fallback.
"""

from .errors import ConfigError, DegenerateSampleError, FormatError, RegistrationError  # noqa: F401
from .records import (DescribedFeatures, DescriptorConfig, FeaturePoint, IntensityImage, MatcherConfig,  # noqa: F401
                      MatchPair, RampedImage, RansacConfig, RegistrationResult, RigidTransform, ScaleSet,
                      apply_linear_ramp, default_alpha)

__version__ = "0.1.0"


def __getattr__(name):
    # GPU entry points import torch lazily so host-only users stay light
    if name in ("detect_features",):
        from .detector import detect_features
        return detect_features
    if name in ("describe_features", "compute_descriptor"):
        from . import descriptor
        return getattr(descriptor, name)
    if name in ("match_features",):
        from .matcher import match_features
        return match_features
    if name in ("ransac_rigid", "estimate_rigid"):
        from . import registration
        return getattr(registration, name)
    if name in ("PipelineConfig", "prepare_image", "register_prepared", "prepare_batch"):
        from . import pipeline
        return getattr(pipeline, name)
    raise AttributeError(name)
