"""CPU-side checks of the C ABI: libfbs.so builds for sm_100a, loads, exports
every function include/fbs.h declares, and rejects bad parameters before
touching the device (no compute call here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1807_02044_b200 import build
    path = build.build()
    import paper_1807_02044_b200 as fbs
    return fbs.load_library(path)


def header_functions():
    txt = open(os.path.join(ROOT, "include", "fbs.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fbs_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    import paper_1807_02044_b200 as fbs
    names = header_functions()
    assert len(names) >= 10
    assert sorted(names) == sorted(fbs.EXPORTS)
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", fbs.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_built_for_sm100a():
    import paper_1807_02044_b200 as fbs
    out = subprocess.run(["cuobjdump", "--list-elf", fbs.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def sass_of(function: str) -> str:
    import paper_1807_02044_b200 as fbs
    out = subprocess.run(["cuobjdump", "-sass", fbs.LIB_PATH], capture_output=True, text=True).stdout
    parts = re.split(r"\n\s*Function : ", out)
    for p in parts:
        if p.startswith(function):
            return p
    raise AssertionError(f"{function} not in the SASS of libfbs.so")


def test_sass_uses_ffma2_tma_dp4a():
    """The fused warp-specialised kernel (radius 4): the aggregation stream issues
    FFMA2 with a broadcast scalar weight (a cost-row loop whose body feeds 2 output
    rows x 4 px x 9 taps x 2 disparity pairs), the cost rows are staged by TMA
    (UTMALDG), the 3x3 dot products use DP4A and the hand-over between producer
    and consumer warps uses mbarriers (SYNCS)."""
    out = sass_of("_ZN3fbs8k_fbs_wsILi4ELb0EEEvNS_8WalkArgsE")
    assert out.count("FFMA2") >= 2 * 4 * 9 * 2
    assert "SYNCS" in out
    assert re.search(r"FFMA2 R\d+, R\d+\.F32, R\d+\.F32x2", out)
    assert "UTMALDG" in out
    assert "IDP.4A" in out or "IDP4A" in out


@pytest.mark.parametrize("args,code", [
    ((2, 10, 0, 5, 1, 1.0, 1.0), -3),
    ((10, 2, 0, 5, 1, 1.0, 1.0), -3),
    ((10, 10, -1, 5, 1, 1.0, 1.0), -2),
    ((10, 10, 5, 5, 1, 1.0, 1.0), -2),
    ((10, 10, 0, 5, -1, 1.0, 1.0), -2),
    ((10, 10, 0, 5, 1, 0.0, 1.0), -2),
    ((10, 10, 0, 5, 1, 1.0, float("nan")), -2),
    ((10, 10, 0, 5, 11, 5.0, 40.0), -4),  # radius > FBS_MAX_RADIUS
    ((10, 10, 0, 5, 4, 5.0, 10.0), -4),   # smallest tap weight < 2^-124 (R#13)
    ((10, 10, 0, 5, 3, 0.7, 32.0), -4),
])
def test_create_rejects_bad_params(lib, args, code):
    h = lib.fbs_create(*args)
    assert not h
    assert lib.fbs_last_error().decode().startswith("fbs_create")


def test_null_handle_calls_fail_cleanly(lib):
    assert lib.fbs_compute(None, None, None, None, None) == -1
    assert lib.fbs_compute_rows(None, None, None, 0, 1, None, None) == -1
    assert lib.fbs_stats(None, None) == -1
    assert lib.fbs_compute_keys(None, None, None, 0, 1, None, None, None, None) == -1
    assert lib.fbs_finalize_keys(10, 10, 0, 5, None, None, None, None, None) == -1
    assert lib.fbs_suggest_ranges(None, None, 2, None, None, None) == -1
    assert lib.fbs_compute_ranged(None, None, None, None, None, None, None) == -1
    lib.fbs_destroy(None)


@pytest.mark.parametrize("args", [
    (10, 10, 0, 5, 1, 5.0, 40.0, 2),          # unknown path
    (10, 10, 0, 5, 7, 5.0, 40.0, 1),          # radius > 6 on the fused path
])
def test_create_ex_rejects(lib, args):
    assert not lib.fbs_create_ex(*args)
    assert lib.fbs_last_error().decode().startswith("fbs_create")


@pytest.mark.parametrize("rows", [(-1, 5), (5, 5), (3, 11)])
def test_create_band_rejects_bad_rows(lib, rows):
    assert not lib.fbs_create_band(10, 10, 0, 5, 1, 5.0, 40.0, 0, *rows)
    assert lib.fbs_last_error().decode().startswith("fbs_create_band")


def test_binding_fails_loudly_without_library(tmp_path):
    import paper_1807_02044_b200 as fbs
    saved = fbs._lib
    fbs._lib = None
    try:
        with pytest.raises(ImportError):
            fbs.load_library(str(tmp_path / "missing.so"))
    finally:
        fbs._lib = saved
