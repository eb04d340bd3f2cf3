"""Whole-pipeline pins for the oracle: the literal brute force on tiny pairs,
known-shift random-dot pairs (exact disparity recovery, derived from
Eq.(1),(6),(9),(10)), and sampled-pixel evaluation == full frame."""
import numpy as np
import pytest

import brute
import stereo_synth as synth

SENT = -2.0


def test_pipeline_matches_brute_force(oracle_lib):
    rng = np.random.default_rng(30)
    for t in range(12):
        H, W = int(rng.integers(5, 13)), int(rng.integers(8, 15))
        d_min = int(rng.integers(0, 2)); d_max = d_min + int(rng.integers(2, 5))
        rho = int(rng.integers(1, 3))
        if t % 2:
            L, R = synth.random_dot(W, H, int(rng.integers(d_min, d_max + 1)), 100 + t)
        else:
            L, R, _, _ = synth.layered(W, H, d_min, d_max, 200 + t, n_rects=2, p_flat=0.4)
        r = oracle_lib.fbs(L, R, d_min, d_max, rho, 3.0, 25.0, threads=1)
        out, dl, dr, al, ar = brute.pipeline(L.tolist(), R.tolist(), d_min, d_max, rho, 3.0, 25.0)
        assert np.max(np.abs(r.agg_l - np.array(al))) < 1e-9
        assert np.max(np.abs(r.agg_r - np.array(ar))) < 1e-9
        bdl = np.array([[-1 if x is None else x for x in row] for row in dl])
        bdr = np.array([[-1 if x is None else x for x in row] for row in dr])
        # brute force and oracle may split only on 1e-9 near-ties
        tie = np.abs(r.best_l - r.second_l) < 1e-9
        assert np.all((r.disp_l == bdl) | tie)
        assert np.array_equal(r.disp_r == -1, bdr == -1)
        same = (r.disp_l == bdl) & ~tie
        assert np.max(np.abs(r.disp - np.array(out))[same], initial=0) < 1e-6


@pytest.mark.parametrize("W,H,s,rho,d_min,d_max", [
    (40, 20, 0, 1, 0, 7), (40, 20, 5, 2, 0, 7), (48, 24, 7, 3, 0, 7),
    (64, 16, 11, 4, 3, 14), (64, 16, 3, 4, 3, 14), (64, 16, 14, 4, 3, 14)])
def test_known_shift_random_dot(oracle_lib, W, H, s, rho, d_min, d_max):
    """I_R(x,y) = I_L(x+s,y): every defined cost at d = s is exactly 1 (up to
    the oracle's rounding), others < 1 a.s., hence d_L = s wherever the d = s
    slice has a defined tap (u >= s + 1 - rho), LRC keeps exactly u >= s and
    rejects u in [s+1-rho, s-1]; round(d^s) = s, and d^s = s at the range
    ends (SURVEY §8(c) 'known-shift random-dot')."""
    L, R = synth.random_dot(W, H, s, 1000 + s)
    r = oracle_lib.fbs(L, R, d_min, d_max, rho, 4.0, 30.0, threads=2)
    us = np.arange(W)[None, :].repeat(H, 0)
    cols = us >= max(0, s + 1 - rho)
    assert np.all(r.disp_l[cols] == s)
    assert np.all(r.valid[us >= s])
    assert not np.any(r.valid[cols & (us < s)])
    ok = r.valid & (us >= s)
    assert np.all(np.rint(r.disp[ok]) == s)
    assert np.all(np.abs(r.disp[ok] - s) < 0.5)
    if s in (d_min, d_max):
        assert np.all(r.disp[ok] == s)


def test_known_shift_sign_convention(oracle_lib):
    """A pair shifted the other way (I_R(x) = I_L(x - s)) must NOT be
    recovered as +s: pins the direction of Eq.(1)'s i_r(x - d, y)."""
    L, R = synth.random_dot(40, 12, 5, 77)
    r_good = oracle_lib.fbs(L, R, 0, 9, 2, 4.0, 30.0)
    r_flip = oracle_lib.fbs(R[:, ::-1].copy(), L[:, ::-1].copy(), 0, 9, 2, 4.0, 30.0)
    assert (r_good.disp_l[:, 8:] == 5).all()
    assert (r_flip.disp_l[:, 8:] == 5).all()  # mirrored pair is again a +5 shift
    Lr, Rr = R, L  # swapped without mirroring: true disparity is -5, outside [0, 9]
    r_bad = oracle_lib.fbs(Lr, Rr, 0, 9, 2, 4.0, 30.0)
    assert (r_bad.disp_l[:, 8:] != 5).mean() > 0.9


@pytest.mark.parametrize("kind", ["layered", "random_dot"])
def test_fbs_pixels_bit_identical_to_full_frame(oracle_lib, kind):
    cfg = synth.CONFIGS["synthetic"]
    if kind == "layered":
        L, R, _, _ = synth.layered(cfg.W, cfg.H, cfg.d_min, cfg.d_max, cfg.seed, p_flat=0.3)
    else:
        L, R = synth.random_dot(cfg.W, cfg.H, 7, cfg.seed)
    full = oracle_lib.fbs(L, R, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r)
    rng = np.random.default_rng(31)
    us = rng.integers(0, cfg.W, 300); vs = rng.integers(0, cfg.H, 300)
    us[:4] = [0, cfg.W - 1, 0, cfg.W - 1]; vs[:4] = [0, 0, cfg.H - 1, cfg.H - 1]
    px = oracle_lib.fbs_pixels(L, R, cfg.d_min, cfg.d_max, cfg.radius, cfg.gamma_d, cfg.gamma_r,
                               us, vs, columns=True)
    assert np.array_equal(px.disp, full.disp[vs, us])
    assert np.array_equal(px.disp_l, full.disp_l[vs, us])
    assert np.array_equal(px.agg_col_l, full.agg_l[vs, us])
    ok = px.disp_l >= 0
    xr = us - px.disp_l
    inside = ok & (xr >= 0)
    assert np.array_equal(px.disp_r_at[inside], full.disp_r[vs[inside], xr[inside]])


def test_layered_textureless_produces_sentinels(oracle_lib):
    L, R, _, _ = synth.layered(60, 40, 0, 9, 5, n_rects=3, p_flat=1.0)
    r = oracle_lib.fbs(L, R, 0, 9, 2, 5.0, 32.0)
    # all layers constant: only layer edges carry texture
    assert (r.cost_l == SENT).mean() > 0.5
    assert (r.disp_l == -1).any()
