"""CPU checks of the C-ABI boundary: the library loads, exports exactly the
symbols include/peakstitch_b200.h declares, and its host-side validation /
planning (no GPU needed) follows the reference's rules."""

import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2405_08578_b200 import _lib
from paper_2405_08578_b200.errors import ConfigError, RegistrationError

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "peakstitch_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^PS_API\s+[\w\s\*]+?\b(ps_\w+)\(", txt, flags=re.M)))


def test_library_loads_and_reports_version():
    assert _lib.lib().ps_abi_version() == _lib.ABI_VERSION == 6


def test_every_declared_symbol_is_exported():
    syms = declared_symbols()
    assert len(syms) >= 13
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(ps_\w+)", out))
    assert set(syms) <= exported, set(syms) - exported
    assert set(SIG for SIG in _lib.SIGNATURES) == set(syms)


def test_library_is_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def plan(nr, nc, scales, dedupe=1, batch=1):
    cap, ws = C.c_int64(), C.c_size_t()
    st = _lib.lib().ps_detect_plan(batch, nr, nc, _lib.int32_array(scales), len(scales), dedupe, C.byref(cap),
                                   C.byref(ws))
    return st, cap.value, ws.value


@pytest.mark.parametrize("nr,nc,scales,expect", [
    (768, 1024, (16, 32, 64), 6144),          # C1: nested -> L_min only
    (1600, 2688, (8, 16, 32, 64, 128), 134400),  # C2
    (1600, 2688, (32, 64, 128), 8400),        # C3
    (8192, 8192, (36,), 103968),              # C4 (L = 36)
    (1080, 1920, (16, 32, 64), 16320),        # C5
])
def test_detect_plan_capacity_matches_count_law(nr, nc, scales, expect):
    st, cap, ws = plan(nr, nc, scales)
    assert st == 0 and cap == expect and ws == 0


def test_detect_plan_raw_capacity_without_dedupe():
    from paper_2405_08578_b200.records import window_count
    st, cap, _ = plan(70, 83, (8, 16, 32), dedupe=0)
    assert st == 0 and cap == sum(2 * window_count(70, 83, s) for s in (8, 16, 32))
    st, cap, ws = plan(300, 400, (32, 40), dedupe=1)  # non-nested: both scales evaluated
    assert st == 0 and cap == 2 * (window_count(300, 400, 32) + window_count(300, 400, 40)) and ws > 0


@pytest.mark.parametrize("scales", [(4, 8, 16), (16, 16), (32, 16), (), (8, 16384)])
def test_detect_plan_rejects_bad_scale_sets(scales):
    st, _, _ = plan(8192, 8192, scales) if scales else (_lib.lib().ps_detect_plan(1, 64, 64, None, 0, 1, None,
                                                                                     None), 0, 0)
    assert st in (_lib.PS_ERR_CONFIG, _lib.PS_ERR_ARGUMENT)
    if scales:
        with pytest.raises(ConfigError):
            _lib.check(st)


def test_status_mapping():
    with pytest.raises(RegistrationError):
        _lib.check(_lib.PS_ERR_REGISTRATION)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.PS_ERR_CUDA)


def test_ransac_rejects_too_few_pairs_before_any_launch():
    L = _lib.lib()
    before = L.ps_kernel_launches()
    st = L.ps_ransac_rigid(None, None, 5, None, 100, 3.0, 8, None, None, None, None, None, 0, None)
    assert st == _lib.PS_ERR_REGISTRATION
    assert L.ps_ransac_rigid(None, None, 50, None, 0, 3.0, 8, None, None, None, None, None, 0, None) == \
        _lib.PS_ERR_CONFIG
    assert L.ps_kernel_launches() == before


def test_match_plan_and_config_errors():
    L = _lib.lib()
    ws = C.c_size_t()
    assert L.ps_match_plan(6144, 6144, 128, 0, 0, C.byref(ws)) == 0 and ws.value > 0
    assert L.ps_match_plan(10, 10, 128, 7, 0, C.byref(ws)) == _lib.PS_ERR_CONFIG
    cnt = C.c_int64()
    assert L.ps_match(None, 1, None, 1, 128, 0, 0.0, 0, None, None, None, C.byref(cnt), 1, None, 0, None) == \
        _lib.PS_ERR_CONFIG


def test_placement_struct_layout_matches_header():
    """ps_placement (include/peakstitch_b200.h): natural C alignment, 80 bytes."""
    P = _lib.PlacementC
    assert C.sizeof(P) == 80
    offs = {name: getattr(P, name).offset for name, _ in P._fields_}
    assert offs["row_pitch"] == 40 and offs["cos_t"] == 48 and offs["t_y"] == 72


def test_warp_and_blend_rejects_unknown_modes_before_any_launch():
    L = _lib.lib()
    arr = (_lib.PlacementC * 1)()
    assert L.ps_warp_and_blend(arr, 0, 4, 4, 0, 0, 7, 0, None, None, None) == _lib.PS_ERR_VALUE
    assert L.ps_warp_and_blend(arr, 0, 4, 4, 0, 0, 0, 9, None, None, None) == _lib.PS_ERR_VALUE


def test_match_plan_strategy_flags():
    """Path flags are explicit per call (no environment switches); the extra
    ratio strategy plans; contradictory or unknown flags are rejected."""
    L, ws = _lib.lib(), C.c_size_t()
    for strat in (_lib.PS_MATCH_NEAREST, _lib.PS_MATCH_THRESHOLD_ALL, _lib.PS_MATCH_RATIO,
                  _lib.PS_MATCH_NEAREST | _lib.PS_MATCH_FORCE_EXACT, _lib.PS_MATCH_NEAREST | _lib.PS_MATCH_FORCE_TC):
        assert L.ps_match_plan(1000, 900, 128, strat, 1000, C.byref(ws)) == 0, strat
    assert L.ps_match_plan(10, 10, 128, _lib.PS_MATCH_FORCE_EXACT | _lib.PS_MATCH_FORCE_TC, 10, C.byref(ws)) == 1
    assert L.ps_match_plan(10, 10, 128, 3, 10, C.byref(ws)) == 1
    assert L.ps_match_plan(10, 10, 128, 0x400, 10, C.byref(ws)) == 1
    # tensor-core workspace only when the TC path will run
    exact, tc = C.c_size_t(), C.c_size_t()
    L.ps_match_plan(64, 64, 128, _lib.PS_MATCH_NEAREST, 64, C.byref(exact))
    L.ps_match_plan(64, 64, 128, _lib.PS_MATCH_NEAREST | _lib.PS_MATCH_FORCE_TC, 64, C.byref(tc))
    assert tc.value > exact.value


def test_library_reads_no_environment():
    """The product library has no hidden getenv switches (ADVICE/VERDICT r1):
    every getenv in csrc/ sits inside an ``#ifdef PS_DIAG`` block (diagnostic
    builds only; the static CUDA runtime's own getenv is not ours)."""
    csrc = os.path.join(REPO, "paper_2405_08578_b200", "csrc")
    for name in sorted(os.listdir(csrc)):
        if not name.endswith((".cu", ".cuh")):
            continue
        depth = []  # stack of "is this #if a PS_DIAG guard"
        for ln, line in enumerate(open(os.path.join(csrc, name)), 1):
            t = line.strip()
            if t.startswith("#if"):
                depth.append("PS_DIAG" in t)
            elif t.startswith("#endif"):
                depth.pop()
            elif "getenv(" in t and not t.startswith("//"):
                assert any(depth), f"{name}:{ln} reads the environment outside #ifdef PS_DIAG"
