"""CPU oracle for the fast bilateral stereo (FBS) hot path — TEST INFRASTRUCTURE.

This package is the plain, slow, double-precision definition of what the B200
path computes (Eq.(1)-(3), (6)-(10); see oracle/fbs_oracle.c for the
per-function citations).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  It
shares no code with ``paper_1807_02044_b200`` and never imports it.

Parity status per function (DESIGN.md §4 lists the pins):
  block_stats, ncc, cost_volumes  pinned (tests/test_oracle_cost.py)
  weights, aggregate              pinned (tests/test_oracle_aggregate.py)
  wta, lrc, subpixel              pinned (tests/test_oracle_select.py)
  fbs (whole pipeline)            pinned on known-shift random-dot pairs and
                                  against the literal brute force
                                  (tests/test_oracle_pipeline.py); on general
                                  natural-like scenes beyond those: parity
                                  unpinned (no reference values exist).
  fbs_pixels                      pinned against fbs (bit-identical).
  ranged.* (sparse search range)  pinned (tests/test_oracle_ranged.py): reduces to
                                  fbs with full ranges; closed forms; known shift.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

SENT = -2.0
INVALID = -1

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fbs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc: -O2, no FP contraction, no fast-math."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
             "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I = ctypes.c_int
        Dd = ctypes.c_double
        _lib.oracle_block_stats.argtypes = [P, I, I, P, P, P]
        _lib.oracle_ncc_at.argtypes = [P, P, I, I, I, I, I]
        _lib.oracle_ncc_at.restype = Dd
        _lib.oracle_cost_volumes.argtypes = [P, P, I, I, I, I, P, P, I]
        _lib.oracle_spatial_weights.argtypes = [I, Dd, P]
        _lib.oracle_range_weights.argtypes = [Dd, P]
        _lib.oracle_aggregate.argtypes = [P, P, I, I, I, I, Dd, Dd, P, I]
        _lib.oracle_wta.argtypes = [P, I, I, I, I, P, P, P]
        _lib.oracle_lrc.argtypes = [P, P, I, I, P]
        _lib.oracle_subpixel.argtypes = [P, P, P, I, I, I, I, P, P]
        _lib.oracle_fbs.argtypes = [P, P, I, I, I, I, I, Dd, Dd, I] + [P] * 11
        _lib.oracle_fbs.restype = I
        _lib.oracle_fbs_pixels.argtypes = [P, P, I, I, I, I, I, Dd, Dd, I, P, P, I] + [P] * 6
        _lib.oracle_fbs_pixels.restype = I
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _img(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint8)
    assert a.ndim == 2
    return a


def default_threads() -> int:
    return os.cpu_count() or 1


# --------------------------------------------------------------------------
# Stage-level functions (each mirrors one C function; see its citation).

def block_stats(img):
    """Eq.(2)(3): (mu, sigma, defined) per pixel; border pixels undefined."""
    img = _img(img)
    H, W = img.shape
    mu = np.zeros((H, W)); sg = np.zeros((H, W)); df = np.zeros((H, W), np.uint8)
    _load().oracle_block_stats(_p(img), W, H, _p(mu), _p(sg), _p(df))
    return mu, sg, df.astype(bool)


def ncc_at(left, right, u: int, v: int, d: int) -> float:
    """Eq.(1) at one (u,v,d) from the raw images; SENT when undefined."""
    left, right = _img(left), _img(right)
    H, W = left.shape
    return float(_load().oracle_ncc_at(_p(left), _p(right), W, H, u, v, d))


def cost_volumes(left, right, d_min: int, d_max: int, threads: int = 1):
    """Twin cost volumes: arrays [H, W, D], SENT where undefined."""
    left, right = _img(left), _img(right)
    H, W = left.shape
    D = d_max - d_min + 1
    cl = np.empty((H, W, D)); cr = np.empty((H, W, D))
    _load().oracle_cost_volumes(_p(left), _p(right), W, H, d_min, d_max, _p(cl), _p(cr), threads)
    return cl, cr


def spatial_weights(rho: int, gamma_d: float) -> np.ndarray:
    """Eq.(7): [(2rho+1), (2rho+1)] indexed [dy+rho, dx+rho]."""
    K1 = 2 * rho + 1
    wd = np.empty((K1, K1))
    _load().oracle_spatial_weights(rho, float(gamma_d), _p(wd))
    return wd


def range_weights(gamma_r: float) -> np.ndarray:
    """Eq.(8): [256] indexed by |delta intensity|."""
    wr = np.empty(256)
    _load().oracle_range_weights(float(gamma_r), _p(wr))
    return wr


def aggregate(cost, guide, rho: int, gamma_d: float, gamma_r: float, threads: int = 1):
    """Eq.(6) on a [H, W, D] volume guided by ``guide`` (uint8 [H, W])."""
    cost = np.ascontiguousarray(cost, dtype=np.float64)
    guide = _img(guide)
    H, W, D = cost.shape
    assert guide.shape == (H, W)
    out = np.empty_like(cost)
    _load().oracle_aggregate(_p(cost), _p(guide), W, H, D, rho, float(gamma_d), float(gamma_r),
                             _p(out), threads)
    return out


def wta(agg, d_min: int):
    """WTA: (disp int32 [H,W], best, second); INVALID = -1."""
    agg = np.ascontiguousarray(agg, dtype=np.float64)
    H, W, D = agg.shape
    disp = np.empty((H, W), np.int32); best = np.empty((H, W)); second = np.empty((H, W))
    _load().oracle_wta(_p(agg), W, H, d_min, d_min + D - 1, _p(disp), _p(best), _p(second))
    return disp, best, second


def lrc(disp_l, disp_r) -> np.ndarray:
    """Eq.(9) with tolerance 1: bool mask of LRC-valid left pixels."""
    dl = np.ascontiguousarray(disp_l, dtype=np.int32)
    dr = np.ascontiguousarray(disp_r, dtype=np.int32)
    H, W = dl.shape
    out = np.empty((H, W), np.uint8)
    _load().oracle_lrc(_p(dl), _p(dr), W, H, _p(out))
    return out.astype(bool)


def subpixel(agg_l, disp_l, valid, d_min: int):
    """Eq.(10): (disp_s float64 [H,W] with -1 for invalid, denominators)."""
    agg_l = np.ascontiguousarray(agg_l, dtype=np.float64)
    H, W, D = agg_l.shape
    dl = np.ascontiguousarray(disp_l, dtype=np.int32)
    vm = np.ascontiguousarray(valid, dtype=np.uint8)
    out = np.empty((H, W)); den = np.empty((H, W))
    _load().oracle_subpixel(_p(agg_l), _p(dl), _p(vm), W, H, d_min, d_min + D - 1, _p(out), _p(den))
    return out, den


@dataclass
class FbsResult:
    cost_l: np.ndarray | None
    cost_r: np.ndarray | None
    agg_l: np.ndarray | None
    agg_r: np.ndarray | None
    disp_l: np.ndarray
    disp_r: np.ndarray
    valid: np.ndarray
    disp: np.ndarray
    best_l: np.ndarray
    second_l: np.ndarray
    sub_den: np.ndarray


def fbs(left, right, d_min: int, d_max: int, rho: int, gamma_d: float, gamma_r: float,
        threads: int | None = None, volumes: bool = True) -> FbsResult:
    """Whole method (Fig. 1 order).  ``volumes=False`` skips exporting the
    four [H,W,D] volumes (they are still computed internally)."""
    left, right = _img(left), _img(right)
    H, W = left.shape
    D = d_max - d_min + 1
    th = threads or default_threads()
    vol = (lambda: np.empty((H, W, D))) if volumes else (lambda: None)
    cl, cr, al, ar = vol(), vol(), vol(), vol()
    dl = np.empty((H, W), np.int32); dr = np.empty((H, W), np.int32)
    vm = np.empty((H, W), np.uint8); ds = np.empty((H, W))
    bl = np.empty((H, W)); sl = np.empty((H, W)); sd = np.empty((H, W))
    rc = _load().oracle_fbs(_p(left), _p(right), W, H, d_min, d_max, rho, float(gamma_d),
                            float(gamma_r), th, _p(cl), _p(cr), _p(al), _p(ar), _p(dl), _p(dr),
                            _p(vm), _p(ds), _p(bl), _p(sl), _p(sd))
    if rc != 0:
        raise ValueError(f"oracle_fbs rejected its arguments (rc={rc})")
    return FbsResult(cl, cr, al, ar, dl, dr, vm.astype(bool), ds, bl, sl, sd)


@dataclass
class PixelResult:
    disp: np.ndarray
    disp_l: np.ndarray
    disp_r_at: np.ndarray
    best_l: np.ndarray
    second_l: np.ndarray
    sub_den: np.ndarray
    agg_col_l: np.ndarray | None


def fbs_pixels(left, right, d_min: int, d_max: int, rho: int, gamma_d: float, gamma_r: float,
               us, vs, threads: int | None = None, columns: bool = False) -> PixelResult:
    """The same method evaluated only at pixels (us[i], vs[i]) (for frames too
    large to materialise; bit-identical to :func:`fbs` at those pixels)."""
    left, right = _img(left), _img(right)
    H, W = left.shape
    D = d_max - d_min + 1
    us = np.ascontiguousarray(us, dtype=np.int32); vs = np.ascontiguousarray(vs, dtype=np.int32)
    n = us.size
    assert vs.size == n
    assert np.all((us >= 0) & (us < W) & (vs >= 0) & (vs < H))
    ds = np.empty(n); dl = np.empty(n, np.int32); dr = np.empty(n, np.int32)
    bl = np.empty(n); sl = np.empty(n); sd = np.empty(n)
    col = np.empty((n, D)) if columns else None
    rc = _load().oracle_fbs_pixels(_p(left), _p(right), W, H, d_min, d_max, rho, float(gamma_d),
                                   float(gamma_r), n, _p(us), _p(vs), threads or default_threads(),
                                   _p(ds), _p(dl), _p(dr), _p(bl), _p(sl), _p(sd), _p(col))
    if rc != 0:
        raise ValueError(f"oracle_fbs_pixels rejected its arguments (rc={rc})")
    return PixelResult(ds, dl, dr, bl, sl, sd, col)
