"""Pins for the oracle's WTA, LRC and parabola subpixel stages."""
import json
import os

import numpy as np
import pytest

import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
SENT = -2.0


def test_wta_worked_example(oracle_lib):
    g = GOLD["wta_column"]
    agg = np.array(g["column"], dtype=np.float64).reshape(1, 1, -1)
    disp, best, second = oracle_lib.wta(agg, g["d_min"])
    assert disp[0, 0] == g["expected"] and best[0, 0] == 0.9 and second[0, 0] == 0.1


def test_wta_all_sentinel_and_ties(oracle_lib):
    agg = np.full((1, 3, 5), SENT)
    agg[0, 1] = [0.1, 0.7, 0.3, 0.7, 0.2]      # tie -> smaller d
    agg[0, 2] = [SENT, 0.4, SENT, 0.4, 0.9]
    disp, best, second = oracle_lib.wta(agg, 3)
    assert disp[0, 0] == -1
    assert disp[0, 1] == 3 + 1 and second[0, 1] == 0.7
    assert disp[0, 2] == 3 + 4 and second[0, 2] == 0.4


def test_wta_matches_brute_on_random_volume(oracle_lib):
    rng = np.random.default_rng(20)
    agg = np.round(rng.uniform(-1, 1, (12, 12, 9)), 1)  # rounding creates ties
    agg[rng.random(agg.shape) < 0.15] = SENT
    disp, _, _ = oracle_lib.wta(agg, 2)
    for v in range(12):
        for u in range(12):
            b = brute.wta(agg[v, u].tolist(), 2)
            assert disp[v, u] == (-1 if b is None else b)
            if b is not None:  # no d' strictly better
                assert np.all(agg[v, u][agg[v, u] != SENT] <= agg[v, u, b - 2])


def test_lrc_worked_examples(oracle_lib):
    for case in GOLD["lrc"]["cases"]:
        W = 12
        dl = np.full((1, W), -1, np.int32); dr = np.full((1, W), -1, np.int32)
        u = 9
        dl[0, u] = case["dl"]; dr[0, u - case["dl"]] = case["dr"]
        assert oracle_lib.lrc(dl, dr)[0, u] == case["valid"]


def test_lrc_out_of_image_and_invalid(oracle_lib):
    dl = np.array([[3, 3, 0, -1, 1]], np.int32)
    dr = np.array([[3, -1, 3, 3, 3]], np.int32)
    ok = oracle_lib.lrc(dl, dr)[0]
    # u=0,1: u-d < 0 ; u=2: dr[2]=3 vs 0 -> |0-3|>1 ; u=3: dl invalid ; u=4: dr[3]=3 vs 1 -> invalid
    assert list(ok) == [False, False, False, False, False]
    dr2 = np.array([[3, 2, 0, 3, 3]], np.int32)  # |0-3|,|0-2| > 1; |0-0| ok; |0-3|; |1-3| > 1
    assert list(oracle_lib.lrc(np.array([[0, 0, 0, 0, 1]], np.int32), dr2)[0]) == [False, False, True, False, False]


def _one_column(c3, d=5, D=11):
    agg = np.full((1, 1, D), 0.0)
    agg[0, 0, d - 1: d + 2] = c3
    return agg


def test_subpixel_worked_examples(oracle_lib):
    for case in GOLD["subpixel"]["cases"]:
        agg = _one_column(case["c"])
        ds, _ = oracle_lib.subpixel(agg, np.array([[5]], np.int32), np.array([[True]]), 0)
        assert ds[0, 0] == pytest.approx(5 + case["delta"], abs=1e-15)


def test_subpixel_parabola_closed_form(oracle_lib):
    """Samples of k - a(x - x0)^2 at x = -1, 0, 1 give the vertex x0 exactly
    (Eq.(10) is the vertex of the parabola through three points)."""
    rng = np.random.default_rng(21)
    for _ in range(2000):
        x0 = rng.uniform(-0.5, 0.5); a = rng.uniform(0.01, 2); k = rng.uniform(-1, 1)
        c3 = [k - a * (x - x0) ** 2 for x in (-1, 0, 1)]
        ds, _ = oracle_lib.subpixel(_one_column(c3), np.array([[5]], np.int32), np.array([[True]]), 0)
        assert ds[0, 0] == pytest.approx(5 + x0, abs=1e-12)


def test_subpixel_strict_max_bound(oracle_lib):
    """|d^s - d| <= 0.5 on 1e4 random strict-max triples; exact on
    symmetric triples."""
    rng = np.random.default_rng(22)
    n = 10000
    c0 = rng.uniform(-1, 1, n)
    cm = c0 - rng.uniform(1e-6, 1, n); cp = c0 - rng.uniform(1e-6, 1, n)
    agg = np.zeros((1, n, 3)); agg[0, :, 0] = cm; agg[0, :, 1] = c0; agg[0, :, 2] = cp
    ds, _ = oracle_lib.subpixel(agg, np.ones((1, n), np.int32), np.ones((1, n), bool), 0)
    assert np.all(np.abs(ds - 1) < 0.5)
    agg[0, :, 2] = cm
    ds, _ = oracle_lib.subpixel(agg, np.ones((1, n), np.int32), np.ones((1, n), bool), 0)
    assert np.all(ds == 1.0)


def test_subpixel_boundary_and_sentinel(oracle_lib):
    agg = np.array([[[0.9, 0.5, 0.1, SENT, 0.3, 0.8]]])
    for d, expect in [(0, 0.0), (5, 5.0), (4, 4.0), (2, 2.0)]:  # boundary d / SENT neighbour
        ds, _ = oracle_lib.subpixel(agg, np.array([[d]], np.int32), np.array([[True]]), 0)
        assert ds[0, 0] == expect
    ds, _ = oracle_lib.subpixel(agg, np.array([[1]], np.int32), np.array([[False]]), 0)
    assert ds[0, 0] == -1.0
