"""Oracle of the sparse search range (NEXT-4) — TEST INFRASTRUCTURE.

PAPER.md §5, future work: "use a group of reliable feature points to
suggest the search range for their neighbours.  Then, only the correlation costs
around the suggested search range are calculated and the bilateral filtering is
performed only on the space around the calculated disparities."  The paper gives
no algorithm; R#31-R#33 fix the reading implemented here:

  R#31 feature points = LRC-valid pixels of a seed disparity map (e.g. the
       previous frame of a stream, or a cheaper pass); "their neighbours" = the
       pixels of the same T x T tile (T = 16, frame-anchored); the suggested
       range of a tile = [floor(min seed) - m, ceil(max seed) + m] over the tile's
       seeds, clipped to [d_min, d_max]; a tile without seeds keeps the full
       range.  The right image's seeds are the left seeds forward-warped
       (x_r = x - round(s)), the same tile rule giving its ranges.
  R#32 the aggregated cost c_agg(p, d) is Eq.(6) unchanged (it does not depend
       on which other d are evaluated); the WTA of pixel p runs over
       its suggested range only: d*(p) = argmax_{d in [lo(p), hi(p)]} c_agg(p, d),
       ties to the smallest d, no defined cost in range -> INVALID.
  R#33 LRC (Eq.(9)) unchanged on the ranged maps; the parabola (Eq.(10)) only when
       d*-1 and d*+1 both lie in the pixel's range (the range end acts like the
       ends of [d_min, d_max] in R#21).

Only ``tests/`` import this module.  It uses the aggregated volumes of
``oracle.fbs`` (double) and plain numpy loops; it shares no code with
``paper_1807_02044_b200``.  Pins: tests/test_oracle_ranged.py (full ranges reduce
to oracle.fbs exactly; brute force on tiny inputs; known-shift recovery).
"""
from __future__ import annotations

import math

import numpy as np

TILE = 16
SENT = -2.0
INVALID = -1


def suggest_ranges(seed, d_min: int, d_max: int, margin: int, tile: int = TILE):
    """R#31: per-pixel (lo, hi) int arrays [H, W, 2] for the left and right images
    from a seed map (float [H, W], < 0 = not a feature point)."""
    seed = np.asarray(seed, dtype=np.float64)
    H, W = seed.shape
    ty, tx = -(-H // tile), -(-W // tile)
    lo_l = np.full((ty, tx), np.inf); hi_l = np.full((ty, tx), -np.inf)
    lo_r = np.full((ty, tx), np.inf); hi_r = np.full((ty, tx), -np.inf)
    for y in range(H):
        for x in range(W):
            s = seed[y, x]
            if s < 0:
                continue
            lo_l[y // tile, x // tile] = min(lo_l[y // tile, x // tile], math.floor(s))
            hi_l[y // tile, x // tile] = max(hi_l[y // tile, x // tile], math.ceil(s))
            xr = x - int(math.floor(s + 0.5))
            if 0 <= xr < W:
                lo_r[y // tile, xr // tile] = min(lo_r[y // tile, xr // tile], math.floor(s))
                hi_r[y // tile, xr // tile] = max(hi_r[y // tile, xr // tile], math.ceil(s))
    out = []
    for lo, hi in ((lo_l, hi_l), (lo_r, hi_r)):
        r = np.empty((H, W, 2), np.int32)
        for y in range(H):
            for x in range(W):
                a, b = lo[y // tile, x // tile], hi[y // tile, x // tile]
                if a > b:  # no feature point in the tile: the full range
                    r[y, x] = (d_min, d_max)
                else:
                    r[y, x] = (max(d_min, int(a) - margin), min(d_max, int(b) + margin))
        out.append(r)
    return out[0], out[1]


def wta_ranged(agg, d_min: int, ranges):
    """R#32: ranged WTA of an aggregated volume [H, W, D] (SENT = undefined)."""
    H, W, D = agg.shape
    disp = np.full((H, W), INVALID, np.int32)
    for y in range(H):
        for x in range(W):
            lo, hi = int(ranges[y, x, 0]), int(ranges[y, x, 1])
            best, bv = INVALID, None
            for d in range(max(lo, d_min), min(hi, d_min + D - 1) + 1):
                c = agg[y, x, d - d_min]
                if c == SENT:
                    continue
                if best == INVALID or c > bv:  # strictly greater: ties keep the smaller d
                    best, bv = d, c
            disp[y, x] = best
    return disp


def fbs_ranged(ref, d_min: int, d_max: int, ranges_l, ranges_r):
    """R#32-R#33 on the volumes of an ``oracle.fbs`` result: (disp, disp_l, disp_r,
    sub_den) with disp float64 [H, W] (-1 = INVALID)."""
    agg_l, agg_r = ref.agg_l, ref.agg_r
    H, W, D = agg_l.shape
    dl = wta_ranged(agg_l, d_min, ranges_l)
    dr = wta_ranged(agg_r, d_min, ranges_r)
    disp = np.full((H, W), float(INVALID))
    den_out = np.zeros((H, W))
    for y in range(H):
        for x in range(W):
            d = int(dl[y, x])
            if d == INVALID or x - d < 0:
                continue
            e = int(dr[y, x - d])
            if e == INVALID or abs(d - e) > 1:  # Eq.(9), tolerance 1 (R#17)
                continue
            ds = float(d)
            lo, hi = int(ranges_l[y, x, 0]), int(ranges_l[y, x, 1])
            if d - 1 >= max(lo, d_min) and d + 1 <= min(hi, d_max):
                cm, c0, cp = agg_l[y, x, d - 1 - d_min], agg_l[y, x, d - d_min], agg_l[y, x, d + 1 - d_min]
                if cm != SENT and cp != SENT:
                    den = 2.0 * cm + 2.0 * cp - 4.0 * c0  # Eq.(10)
                    den_out[y, x] = den
                    if abs(den) >= 1e-9:
                        ds = d + min(0.5, max(-0.5, (cm - cp) / den))
            disp[y, x] = ds
    return disp, dl, dr, den_out
