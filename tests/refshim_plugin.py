"""pytest plugin: run the reference's OWN test files with its hot-path entry
points swapped for the B200 drop-ins (the INTEGRATION.md swap, applied to
the installed reference in ``baseline/_ref``).

Loaded with ``-p refshim_plugin`` before the reference's test modules are
collected, so their ``from peakstitch.detector import detect_features``
binds the drop-in.  Swapped:

  peakstitch.detector.detect_features        detector.py:154-172
  peakstitch.descriptor.describe_features    descriptor.py:259-269
  peakstitch.descriptor.compute_descriptor   descriptor.py:219-256
  peakstitch.matcher.match_features          matcher.py:57-95
  peakstitch.registration.ransac_rigid       registration.py:149-203
  peakstitch.registration.estimate_rigid     registration.py:107-131

and the same names inside ``peakstitch.pipeline`` (its callers,
pipeline.py:26-37).  Every swapped call is counted; the counts are written to
``$PS_REFSHIM_COUNTS`` at session end so the calling test can prove the GPU
path ran.  Test infrastructure only.
"""

from __future__ import annotations

import functools
import json
import os

COUNTS: dict = {}


def _counted(name, fn):
    @functools.wraps(fn)
    def wrapper(*a, **k):
        COUNTS[name] = COUNTS.get(name, 0) + 1
        return fn(*a, **k)

    return wrapper


def _swap():
    import peakstitch.descriptor as rdesc
    import peakstitch.detector as rdet
    import peakstitch.matcher as rmat
    import peakstitch.pipeline as rpipe
    import peakstitch.registration as rreg

    from paper_2405_08578_b200 import descriptor, detector, errors, matcher, registration

    assert errors.REFERENCE_CLASSES, "the drop-ins must raise the reference's exception classes"
    table = [
        (rdet, "detect_features", detector.detect_features),
        (rdesc, "describe_features", descriptor.describe_features),
        (rdesc, "compute_descriptor", descriptor.compute_descriptor),
        (rmat, "match_features", matcher.match_features),
        (rreg, "ransac_rigid", registration.ransac_rigid),
        (rreg, "estimate_rigid", registration.estimate_rigid),
    ]
    for mod, name, fn in table:
        wrapped = _counted(name, fn)
        setattr(mod, name, wrapped)
        if hasattr(rpipe, name):
            setattr(rpipe, name, wrapped)


def pytest_configure(config):
    _swap()


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("PS_REFSHIM_COUNTS")
    if path:
        with open(path, "w") as f:
            json.dump(COUNTS, f)
