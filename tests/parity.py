"""GPU <-> oracle comparison rules (BASELINE.json north_star).

  costs, aggregated costs   |gpu - ref| <= 1e-6 |ref| + 1e-6         (sentinel patterns equal)
  integer WTA maps          bit-exact, except logged near-ties: allowed iff
                            agg_ref(p, d_gpu) >= agg_ref(p, d_ref) - 1e-5
  LRC mask                  exact where both maps (and the d_R they read) agree
  subpixel                  |gpu - ref| <= 1e-3 px where d and LRC agree; pixels whose
                            oracle parabola denominator |den| < 1e-3 are logged apart

The aggregated-cost bound is SURVEY §8(c)'s 1e-6 (plus 1e-6 relative).  The
rigorous fp32 worst case of a K-term weighted mean is ~2 K u (u = 2^-24:
2.0e-5 at K = 169); the observed maximum over every GPU parity case is
9.1e-7 (DESIGN.md §4 lists them per case), so the tight bound is the contract.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SENT = -2.0
REL = 1e-6
TIE = 1e-5
SUBPIX = 1e-3
SMALL_DEN = 1e-3


def agg_abs_floor(radius: int) -> float:
    """Absolute part of the aggregated-cost tolerance; radius-independent."""
    return 1e-6


def check_volume(gpu: np.ndarray, ref: np.ndarray, abs_floor: float, name: str):
    gpu = np.asarray(gpu, dtype=np.float64)
    gs, rs = gpu == SENT, ref == SENT
    bad_pattern = np.argwhere(gs != rs)
    assert bad_pattern.size == 0, f"{name}: sentinel pattern differs at {bad_pattern[:5].tolist()}"
    d = np.abs(gpu - ref)[~rs]
    tol = REL * np.abs(ref[~rs]) + abs_floor
    worst = float(np.max(d - tol, initial=-1))
    assert worst <= 0, f"{name}: max excess {worst:.3e} (max abs err {float(d.max()):.3e})"
    return float(d.max(initial=0.0))


@dataclass
class MapReport:
    n: int = 0
    near_ties: int = 0
    cascades: int = 0
    small_den: int = 0
    max_subpix_err: float = 0.0
    notes: list = field(default_factory=list)


def check_int_map(d_gpu: np.ndarray, d_ref: np.ndarray, agg_ref_at, name: str, rep: MapReport):
    """agg_ref_at(idx, d) -> oracle aggregated cost at flat pixel idx, disparity d."""
    d_gpu = np.asarray(d_gpu).ravel(); d_ref = np.asarray(d_ref).ravel()
    diff = np.flatnonzero(d_gpu != d_ref)
    for i in diff:
        g, r = int(d_gpu[i]), int(d_ref[i])
        assert g >= 0 and r >= 0, f"{name}: validity differs at {i}: gpu {g} ref {r}"
        cg, cr = agg_ref_at(i, g), agg_ref_at(i, r)
        assert cg >= cr - TIE, f"{name}: pixel {i} gpu d={g} (c={cg}) vs ref d={r} (c={cr})"
        rep.near_ties += 1
    rep.n += d_gpu.size
    return diff


def check_final(ds_gpu, ds_ref, dl_gpu, dl_ref, dr_gpu, dr_ref, den_ref, W, rep: MapReport,
                tied_left=None):
    """Final subpixel maps; pixels whose decision chain contains a near-tie are cascades."""
    ds_gpu = np.asarray(ds_gpu, np.float64).ravel(); ds_ref = np.asarray(ds_ref).ravel()
    dl_gpu = np.asarray(dl_gpu).ravel(); dl_ref = np.asarray(dl_ref).ravel()
    dr_gpu = np.asarray(dr_gpu).ravel(); dr_ref = np.asarray(dr_ref).ravel()
    den_ref = np.asarray(den_ref).ravel()
    n = ds_ref.size
    idx = np.arange(n)
    u = idx % W
    same_l = dl_gpu == dl_ref
    # the d_R each side read in its LRC
    xr = u - dl_ref
    ok_r = (dl_ref >= 0) & (xr >= 0)
    rd = np.where(ok_r, idx - dl_ref, 0)
    same_r = ~ok_r | (dr_gpu[rd] == dr_ref[rd])
    chain_ok = same_l & same_r
    rep.cascades += int((~chain_ok).sum())
    v_gpu, v_ref = ds_gpu >= 0, ds_ref >= 0
    bad = chain_ok & (v_gpu != v_ref)
    assert not bad.any(), f"LRC differs at {np.flatnonzero(bad)[:5].tolist()}"
    both = chain_ok & v_ref
    small = both & (np.abs(den_ref) < SMALL_DEN) & (np.abs(den_ref) > 0)
    rep.small_den += int(small.sum())
    chk = both & ~small
    err = np.abs(ds_gpu - ds_ref)[chk]
    rep.max_subpix_err = max(rep.max_subpix_err, float(err.max(initial=0.0)))
    assert rep.max_subpix_err <= SUBPIX, f"subpixel error {rep.max_subpix_err}"
    # integer parts must agree even at small denominators (|delta| <= 0.5 on both sides)
    assert np.all(np.abs(ds_gpu - ds_ref)[small] <= 1.0)
