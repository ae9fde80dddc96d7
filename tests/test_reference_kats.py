"""The reference's own known-answer tests, run through the B200 drop-ins.

``tools/install_reference.sh`` installs the unmodified reference into
``baseline/_ref`` (git-ignored; it travels to the GPU box) together with its
test files.  Each test here runs one of those files in a child pytest with
``tests/refshim_plugin.py`` swapping ``detect_features`` /
``describe_features`` / ``compute_descriptor`` / ``match_features`` /
``ransac_rigid`` / ``estimate_rigid`` (and the same names inside
``peakstitch.pipeline``) for this package's GPU implementations, and then
checks that the swapped entry points were really called.

KAT files: test_detector.py:30-211,
test_descriptor.py:34-235, test_matcher.py:27-148, test_registration.py:34-200,
and the callers: test_acceptance.py (criteria 1-6), test_mosaic.py,
test_pipeline_cli.py (stitch_pair / build_pairwise_table through the swap).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "peakstitch_tests")

needs_ref = pytest.mark.skipif(not os.path.isdir(os.path.join(REF_TESTS)),
                               reason="reference not installed (tools/install_reference.sh)")

# entry points each file must drive through the drop-ins
EXPECT = {
    "test_detector.py": {"detect_features"},
    "test_descriptor.py": {"compute_descriptor", "describe_features"},
    "test_matcher.py": {"match_features"},
    "test_registration.py": {"ransac_rigid", "estimate_rigid"},
    "test_acceptance.py": {"detect_features", "compute_descriptor", "ransac_rigid"},
    "test_mosaic.py": {"detect_features", "describe_features", "match_features", "ransac_rigid"},
    "test_pipeline_cli.py": {"detect_features", "describe_features", "match_features", "ransac_rigid"},
}


def _run(fname, tmp_path, plugin=True):
    counts = tmp_path / "counts.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, REF_TESTS, os.path.join(REPO, "tests"), REPO,
                                         env.get("PYTHONPATH", "")])
    env["PS_REFSHIM_COUNTS"] = str(counts)
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-o", "addopts=",
           "--rootdir", REF_TESTS, "-c", os.devnull]
    if plugin:
        cmd += ["-p", "refshim_plugin"]
    cmd.append(os.path.join(REF_TESTS, fname))
    proc = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=1800)
    got = json.loads(counts.read_text()) if counts.exists() else {}
    return proc, got


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("fname", sorted(EXPECT))
def test_reference_kats_through_dropins(fname, tmp_path):
    proc, counts = _run(fname, tmp_path)
    tail = (proc.stdout + proc.stderr)[-4000:]
    assert proc.returncode == 0, f"reference {fname} failed through the drop-ins:\n{tail}"
    missing = {n for n in EXPECT[fname] if counts.get(n, 0) == 0}
    assert not missing, f"{fname}: drop-ins never called: {missing}; counts {counts}"
    print(f"{fname}: {proc.stdout.strip().splitlines()[-1]}; drop-in calls {counts}")


SWAP_SCRIPT = r'''
import numpy as np
import refshim_plugin
refshim_plugin._swap()                      # the INTEGRATION.md swap
from peakstitch import pipeline as P
from peakstitch.imaging import IntensityImage
from peakstitch.registration import RegistrationResult
from paper_2405_08578_b200 import scenes
cfg = P.PipelineConfig(window_min=16, window_max=64, ransac_iters=500)
s1, s2 = scenes.scene(320, 320, 11), scenes.scene(320, 320, 12)   # unrelated images
a, b = (P.prepare_image(IntensityImage(x.astype(float), n), cfg) for x, n in ((s1, "a"), (s2, "b")))
pairs, res, _, _ = P.register_prepared(a, b, cfg, seed=0)
assert res is None, res                    # RegistrationError caught by the reference's except clause
s = scenes.scene(320, 480, 3)
a, b = (P.prepare_image(IntensityImage(x.astype(float), n), cfg) for x, n in ((s[:, :320], "a"), (s[:, 160:], "b")))
pairs, res, _, _ = P.register_prepared(a, b, cfg, seed=0)
assert isinstance(res, RegistrationResult) and res.consensus_size >= 8
assert abs(res.transform.t_x + 160) < 1e-6 and abs(res.transform.t_y) < 1e-6, res.transform
print("swap ok", len(pairs), res.consensus_size, refshim_plugin.COUNTS)
'''


@needs_ref
@pytest.mark.gpu
def test_reference_register_prepared_through_swap(tmp_path):
    """after the swap the reference's register_prepared
    (pipeline.py:204-207) must turn the drop-in's RegistrationError into None."""
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(REPO, "tests"), REPO, env.get("PYTHONPATH", "")])
    proc = subprocess.run([sys.executable, "-c", SWAP_SCRIPT], cwd=str(tmp_path), env=env,
                          capture_output=True, text=True, timeout=900)
    assert proc.returncode == 0, (proc.stdout + proc.stderr)[-4000:]
    assert "swap ok" in proc.stdout


@needs_ref
def test_errors_alias_reference_classes(tmp_path):
    """CPU: with the reference importable, the package's exception classes ARE
    the reference's (errors.py)."""
    code = ("import peakstitch.errors as R, paper_2405_08578_b200.errors as E\n"
            "assert E.REFERENCE_CLASSES\n"
            "assert all(getattr(E, n) is getattr(R, n) for n in "
            "('ConfigError','FormatError','DegenerateSampleError','RegistrationError'))\n"
            "from paper_2405_08578_b200.records import ScaleSet\n"
            "try:\n    ScaleSet((4, 8))\nexcept R.ConfigError:\n    print('ok')\n")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, REPO, env.get("PYTHONPATH", "")])
    proc = subprocess.run([sys.executable, "-c", code], cwd=str(tmp_path), env=env, capture_output=True,
                          text=True, timeout=300)
    assert proc.returncode == 0 and "ok" in proc.stdout, proc.stderr[-2000:]


PLAN_SCRIPT = r'''
import numpy as np
from peakstitch import mosaic as RM
from peakstitch.registration import RigidTransform as RT
from paper_2405_08578_b200 import mosaic as M
from paper_2405_08578_b200.records import RigidTransform as MT
rng = np.random.default_rng(5)
for trial in range(300):
    n = int(rng.integers(2, 10))
    rt, mt = RM.PairwiseTransformTable(n=n), M.PairwiseTransformTable(n=n)
    for a in range(n):
        for b in range(a + 1, n):
            if rng.random() < float(rng.choice([0.15, 0.4, 0.8])):
                th, tx, ty = rng.uniform(-3, 3), rng.uniform(-99, 99), rng.uniform(-99, 99)
                k = int(rng.integers(8, 12))  # few distinct counts: many ties
                rt.set_pair(a, b, RT(th, tx, ty), k)
                mt.set_pair(a, b, MT(th, tx, ty), k)
    ids = [f"i{k}" for k in range(n)]
    rp, rplaced = RM.plan_mosaic(rt, ids)
    mp_, mplaced = M.plan_mosaic(mt, ids)
    assert [(r.reference_id, r.stitched_ids) for r in rp.rounds] == [(r.reference_id, r.stitched_ids) for r in mp_.rounds]
    assert rp.final_unmatched == mp_.final_unmatched
    assert sorted(rplaced) == sorted(mplaced)
    for k in rplaced:
        a, b = rplaced[k], mplaced[k]
        assert (a.theta, a.t_x, a.t_y) == (b.theta, b.t_x, b.t_y), (trial, k)
    for rem in ({0}, set(range(n))):
        assert RM.select_reference(rt, rem) == M.select_reference(mt, rem)
print("plan ok")
'''


@needs_ref
def test_planner_equals_reference_planner(tmp_path):
    """CPU: the inlier-matrix planner (mosaic.plan_mosaic) reproduces the
    reference's plan_mosaic (mosaic.py:130-180) -- rounds, anchors, order,
    unmatched, placements bit for bit -- on 300 random tables with tied
    inlier counts."""
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, REPO, env.get("PYTHONPATH", "")])
    proc = subprocess.run([sys.executable, "-c", PLAN_SCRIPT], cwd=str(tmp_path), env=env, capture_output=True,
                          text=True, timeout=600)
    assert proc.returncode == 0 and "plan ok" in proc.stdout, (proc.stdout + proc.stderr)[-3000:]
