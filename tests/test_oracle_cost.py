"""Pins for the oracle's block statistics and NCC cost volumes (Eq.(1)-(3)).

Every check compares the oracle against something other than itself: the
paper's/SPEC's worked values, exact rational arithmetic, closed-form
invariances of NCC, or the literal brute force in tests/brute.py."""
import json
import math
import os

import numpy as np
import pytest

import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
SENT = -2.0


def test_block_stats_worked_example(oracle_lib):
    g = GOLD["block_stats_3x3"]
    mu, sg, df = oracle_lib.block_stats(np.array(g["image"], np.uint8))
    assert df[1, 1] and not df[0, 0] and not df[2, 2]
    assert mu[1, 1] == pytest.approx(g["mu"], abs=1e-15)
    assert sg[1, 1] == pytest.approx(math.sqrt(g["sigma_squared_times_9"] / 9.0), abs=1e-14)


def test_block_stats_constant_gives_zero_sigma_and_sentinel(oracle_lib):
    v = GOLD["block_stats_constant"]["value"]
    img = np.full((5, 6), v, np.uint8)
    mu, sg, df = oracle_lib.block_stats(img)
    assert np.all(mu[df] == v) and np.all(sg[df] == 0.0)
    cl, cr = oracle_lib.cost_volumes(img, img, 0, 1)
    assert np.all(cl == SENT) and np.all(cr == SENT)


def test_border_undefined(oracle_lib):
    rng = np.random.default_rng(1)
    L = rng.integers(0, 256, (7, 9), dtype=np.uint8)
    cl, cr = oracle_lib.cost_volumes(L, L, 0, 3)
    assert np.all(cl[0] == SENT) and np.all(cl[-1] == SENT)
    assert np.all(cl[:, 0] == SENT) and np.all(cl[:, -1] == SENT)
    # right block centre u-d must be >= 1 (Eq.(1) i_r(x-d, y), block half-width 1)
    for d in range(4):
        assert np.all(cl[:, : d + 1, d] == SENT)


def test_identical_images_d0_is_one(oracle_lib):
    rng = np.random.default_rng(2)
    L = rng.integers(0, 256, (10, 12), dtype=np.uint8)
    cl, _ = oracle_lib.cost_volumes(L, L, 0, 2)
    inner = cl[1:-1, 1:-1, 0]
    assert np.all(np.abs(inner - 1.0) < 1e-12)


@pytest.mark.parametrize("a,b,expected", [(2, 5, 1.0), (1, 7, 1.0), (-1, 255, -1.0)])
def test_affine_invariance(oracle_lib, a, b, expected):
    """NCC is invariant to gain/offset ('more accurate results when the
    intensity difference is involved'): right = a*left + b -> +-1."""
    rng = np.random.default_rng(3)
    L = rng.integers(0, 100, (8, 8), dtype=np.int64)
    R = (a * L + b).astype(np.uint8)
    cl, _ = oracle_lib.cost_volumes(L.astype(np.uint8), R, 0, 0)
    inner = cl[1:-1, 1:-1, 0]
    assert np.all(np.abs(inner - expected) < 1e-12)


def test_range_and_twin_bit_exact(oracle_lib):
    rng = np.random.default_rng(4)
    for _ in range(20):
        H, W = rng.integers(3, 17, 2)
        d_min = int(rng.integers(0, 3)); d_max = d_min + int(rng.integers(1, 6))
        L = rng.integers(0, 256, (H, W), dtype=np.uint8)
        R = rng.integers(0, 256, (H, W), dtype=np.uint8)
        cl, cr = oracle_lib.cost_volumes(L, R, d_min, d_max)
        dfn = cl != SENT
        assert np.all((cl[dfn] >= -1.0) & (cl[dfn] <= 1.0))
        # c at (u,v,d) in the left volume equals (u-d,v,d) in the right one
        n = 0
        for v in range(H):
            for u in range(W):
                for k in range(d_max - d_min + 1):
                    d = d_min + k
                    if cl[v, u, k] != SENT:
                        assert cr[v, u - d, k] == cl[v, u, k]  # bit-exact
                        n += 1
        assert n == int(dfn.sum()) == int((cr != SENT).sum())


def test_cost_matches_brute_force(oracle_lib):
    """SPEC acceptance 1: >=100 random pairs up to 16x16, d_max <= 5,
    both volumes within 1e-6 of the literal brute force (we require 1e-9)."""
    rng = np.random.default_rng(5)
    for t in range(100):
        H, W = (int(x) for x in rng.integers(3, 17, 2))
        d_min = int(rng.integers(0, 2)); d_max = int(rng.integers(d_min + 1, 6))
        L = rng.integers(0, 256, (H, W), dtype=np.uint8)
        if t % 3 == 0:  # low-texture blocks stress cancellation
            L = (200 + rng.integers(0, 3, (H, W))).astype(np.uint8)
        R = rng.integers(0, 256, (H, W), dtype=np.uint8) if t % 2 else np.roll(L, 1, axis=1)
        if t % 5 == 0:
            R[:, : W // 2] = 77  # textureless right region -> sentinels
        cl, cr = oracle_lib.cost_volumes(L, R, d_min, d_max)
        bl, br = brute.cost_volumes(L.tolist(), R.tolist(), d_min, d_max)
        bl, br = np.array(bl), np.array(br)
        assert np.array_equal(cl == SENT, bl == SENT)
        assert np.array_equal(cr == SENT, br == SENT)
        assert np.max(np.abs(cl - bl), initial=0) < 1e-9
        assert np.max(np.abs(cr - br), initial=0) < 1e-9


def test_cost_vs_exact_rational(oracle_lib):
    """Oracle's literal double Eq.(1) vs exact integer arithmetic rounded once:
    within 1e-9 on worst-case low-texture uint8 blocks (R#5)."""
    rng = np.random.default_rng(6)
    worst = 0.0
    for t in range(300):
        base = int(rng.integers(0, 254))
        L = (base + rng.integers(0, 2 + t % 3, (3, 3 + t % 2))).astype(np.uint8)
        R = (int(rng.integers(0, 254)) + rng.integers(0, 2 + t % 2, L.shape)).astype(np.uint8)
        W = L.shape[1]
        for u in range(1, W - 1):
            c = oracle_lib.ncc_at(L, R, u, 1, 0)
            e = brute.ncc_exact(L.tolist(), R.tolist(), u, 1, 0)
            assert (c == SENT) == (e == SENT)
            if c != SENT:
                worst = max(worst, abs(c - e))
    assert worst < 1e-9
