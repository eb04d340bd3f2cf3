"""Pins of the sparse-search-range oracle (oracle/ranged.py, NEXT-4, DESIGN.md
R#31-R#33) against things other than itself: the pinned full-range oracle, closed
forms, and a known-shift recovery."""
import numpy as np
import pytest

import stereo_synth as synth
from oracle import ranged


@pytest.fixture(scope="module")
def scene(oracle_lib):
    W, H, d_min, d_max, rho = 48, 36, 2, 25, 2
    L, R, _, _ = synth.layered(W, H, d_min, d_max, 31, p_flat=0.3)
    ref = oracle_lib.fbs(L, R, d_min, d_max, rho, 5.0, 32.0, threads=1)
    return W, H, d_min, d_max, ref


def full(H, W, d_min, d_max):
    r = np.empty((H, W, 2), np.int32)
    r[..., 0], r[..., 1] = d_min, d_max
    return r


def test_full_ranges_reduce_to_the_oracle(scene):
    """R#32/R#33 with [lo, hi] = [d_min, d_max] everywhere is exactly the pinned
    full-range pipeline (WTA, LRC, subpixel)."""
    W, H, d_min, d_max, ref = scene
    r = full(H, W, d_min, d_max)
    disp, dl, dr, _ = ranged.fbs_ranged(ref, d_min, d_max, r, r)
    assert np.array_equal(dl, ref.disp_l) and np.array_equal(dr, ref.disp_r)
    assert np.array_equal(disp, ref.disp)


def test_single_disparity_ranges(scene):
    """A range [d, d] leaves exactly one candidate: d_L = d wherever c_agg(p, d) is
    defined, INVALID elsewhere; no subpixel (neighbours outside the range)."""
    W, H, d_min, d_max, ref = scene
    d = 9
    r = np.empty((H, W, 2), np.int32)
    r[..., 0] = r[..., 1] = d
    disp, dl, dr, den = ranged.fbs_ranged(ref, d_min, d_max, r, r)
    defined = ref.agg_l[:, :, d - d_min] != ranged.SENT
    assert np.all(dl[defined] == d) and np.all(dl[~defined] == ranged.INVALID)
    ok = disp >= 0
    assert np.all(disp[ok] == d) and np.all(den == 0)


def test_ranged_best_is_the_masked_maximum(scene):
    """The chosen value is the maximum of c_agg over the range (checked as an
    ordering property on random ranges) and enlarging a range never lowers it."""
    W, H, d_min, d_max, ref = scene
    rng = np.random.default_rng(4)
    lo = rng.integers(d_min, d_max + 1, (H, W)); hi = np.minimum(d_max, lo + rng.integers(0, 6, (H, W)))
    r = np.stack([lo, hi], -1).astype(np.int32)
    dl = ranged.wta_ranged(ref.agg_l, d_min, r)
    dl_full = ref.disp_l
    for y in range(H):
        for x in range(W):
            col = ref.agg_l[y, x, lo[y, x] - d_min: hi[y, x] - d_min + 1]
            vals = col[col != ranged.SENT]
            if vals.size == 0:
                assert dl[y, x] == ranged.INVALID
                continue
            v = ref.agg_l[y, x, dl[y, x] - d_min]
            assert v == vals.max() and lo[y, x] <= dl[y, x] <= hi[y, x]
            # the first index reaching the maximum (ties -> smallest d)
            assert dl[y, x] == lo[y, x] + int(np.flatnonzero(col == vals.max())[0])
            if dl_full[y, x] >= 0:
                assert ref.agg_l[y, x, dl_full[y, x] - d_min] >= v


def test_known_shift_recovered_with_a_narrow_range(oracle_lib):
    """Random dot shifted by s: with seeds = s everywhere and margin 2, the
    suggested range [s-2, s+2] contains s and the ranged map equals s wherever
    the full-range oracle finds s (Eq.(1) gives c = 1 there, the maximum)."""
    W, H, s = 40, 24, 7
    L, R = synth.random_dot(W, H, s, 77)
    ref = oracle_lib.fbs(L, R, 0, 15, 2, 5.0, 32.0, threads=1)
    seed = np.full((H, W), float(s))
    rl, rr = ranged.suggest_ranges(seed, 0, 15, 2)
    assert np.all(rl[..., 0] == s - 2) and np.all(rl[..., 1] == s + 2)
    disp, dl, _, _ = ranged.fbs_ranged(ref, 0, 15, rl, rr)
    hit = ref.disp_l == s
    assert hit.mean() > 0.8 and np.all(dl[hit] == s)


def test_suggest_ranges_closed_form():
    """Tiles with seeds get [floor(min) - m, ceil(max) + m] clipped; tiles without
    seeds the full range; the right image's tiles see the seeds at x - round(s)."""
    H, W = 20, 40
    seed = np.full((H, W), -1.0)
    seed[3, 5] = 4.4; seed[10, 12] = 6.6     # tile (0, 0): left range [4-1, 7+1]
    seed[2, 35] = 30.0                       # tile (0, 2): right pixel 35 - 30 = 5 -> right tile (0, 0)
    rl, rr = ranged.suggest_ranges(seed, 0, 31, 1)
    assert tuple(rl[0, 0]) == (3, 8) and tuple(rl[15, 15]) == (3, 8)
    assert tuple(rl[0, 20]) == (0, 31)                       # tile (0, 1): no seed
    assert tuple(rl[0, 39]) == (29, 31)                      # [30-1, 30+1] clipped to 31
    # right tile (0, 0) receives 4.4 -> x 1, 6.6 -> x 5 and 30 -> x 5: [4-1, 30+1] clipped
    assert tuple(rr[0, 0]) == (3, 31)
    assert tuple(rr[0, 39]) == (0, 31)
