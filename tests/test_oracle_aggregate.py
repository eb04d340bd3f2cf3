"""Pins for the oracle's bilateral weights and aggregation (Eq.(6)-(8))."""
import json
import math
import os

import numpy as np
import pytest

import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
SENT = -2.0


def test_weight_worked_examples(oracle_lib):
    g = GOLD["spatial_weight"]
    wd = oracle_lib.spatial_weights(1, g["gamma_d"])
    assert wd[1 + g["dy"], 1 + g["dx"]] == pytest.approx(g["expected"], rel=1e-15)
    assert wd[1, 1] == 1.0
    g = GOLD["range_weight"]
    wr = oracle_lib.range_weights(g["gamma_r"])
    assert wr[g["delta"]] == pytest.approx(g["expected"], rel=1e-15)
    assert wr[0] == 1.0


@pytest.mark.parametrize("rho,gd", [(2, 1.0), (4, 5.0), (6, 3.3)])
def test_spatial_weights_symmetry(oracle_lib, rho, gd):
    wd = oracle_lib.spatial_weights(rho, gd)
    assert np.array_equal(wd, wd.T)
    assert np.array_equal(wd, wd[::-1, :]) and np.array_equal(wd, wd[:, ::-1])
    assert np.all((wd > 0) & (wd <= 1))


@pytest.mark.parametrize("gr", [3.0, 10.0, 32.0, 200.0])
def test_range_weights_monotone(oracle_lib, gr):
    wr = oracle_lib.range_weights(gr)
    nz = wr[wr > 0]
    assert np.all(np.diff(nz) < 0)
    assert np.all(wr <= 1.0)


def test_aggregate_matches_brute_force(oracle_lib):
    """SPEC acceptance 2: >=50 random volumes up to 9x9x6 within 1e-6
    of the literal Eq.(6)-(8) double loop (we require 1e-12)."""
    rng = np.random.default_rng(10)
    for t in range(50):
        H, W, D = (int(rng.integers(1, 10)), int(rng.integers(1, 10)), int(rng.integers(1, 7)))
        rho = int(rng.integers(0, 4))
        gd, gr = float(rng.uniform(0.5, 8)), float(rng.uniform(2, 60))
        cost = rng.uniform(-1, 1, (H, W, D))
        cost[rng.random((H, W, D)) < 0.2] = SENT
        guide = rng.integers(0, 256, (H, W), dtype=np.uint8)
        got = oracle_lib.aggregate(cost, guide, rho, gd, gr)
        ref = np.array(brute.aggregate(cost.tolist(), guide.tolist(), rho, gd, gr))
        assert np.array_equal(got == SENT, ref == SENT)
        assert np.max(np.abs(got - ref), initial=0) < 1e-12


def test_rho0_identity(oracle_lib):
    rng = np.random.default_rng(11)
    cost = rng.uniform(-1, 1, (6, 7, 4)); cost[0, 0, 0] = SENT
    guide = rng.integers(0, 256, (6, 7), dtype=np.uint8)
    got = oracle_lib.aggregate(cost, guide, 0, 5.0, 10.0)
    assert np.array_equal(got, cost)


def test_constant_slice_normalised_weights(oracle_lib):
    """Normalised weights sum to 1 (north_star pin): c == k -> c_agg == k."""
    rng = np.random.default_rng(12)
    cost = np.full((9, 11, 3), 0.5); cost[:, :, 1] = -0.25; cost[:, :, 2] = 1.0
    cost[rng.random(cost.shape) < 0.3] = SENT
    guide = rng.integers(0, 256, (9, 11), dtype=np.uint8)
    got = oracle_lib.aggregate(cost, guide, 3, 4.0, 15.0)
    for k, val in enumerate([0.5, -0.25, 1.0]):
        sl = got[:, :, k]
        assert np.all(np.abs(sl[sl != SENT] - val) < 1e-15)


def test_convex_hull_and_box_limit(oracle_lib):
    rng = np.random.default_rng(13)
    cost = rng.uniform(-1, 1, (8, 8, 2)); cost[rng.random(cost.shape) < 0.1] = SENT
    guide = rng.integers(0, 256, (8, 8), dtype=np.uint8)
    rho = 2
    got = oracle_lib.aggregate(cost, guide, rho, 3.0, 20.0)
    box = oracle_lib.aggregate(cost, guide, rho, 1e9, 1e9)
    for v in range(8):
        for u in range(8):
            for k in range(2):
                win = cost[max(0, v - rho): v + rho + 1, max(0, u - rho): u + rho + 1, k]
                win = win[win != SENT]
                if win.size == 0:
                    assert got[v, u, k] == SENT
                    continue
                assert win.min() - 1e-15 <= got[v, u, k] <= win.max() + 1e-15
                assert abs(box[v, u, k] - win.mean()) < 1e-6


def test_constant_guide_independent_of_gamma_r(oracle_lib):
    rng = np.random.default_rng(14)
    cost = rng.uniform(-1, 1, (7, 9, 3))
    guide = np.full((7, 9), 90, np.uint8)
    a = oracle_lib.aggregate(cost, guide, 2, 2.0, 3.0)
    b = oracle_lib.aggregate(cost, guide, 2, 2.0, 300.0)
    assert np.array_equal(a, b)


def test_weight_symmetry_pq(oracle_lib):
    """w(p,q) = ω_d ω_r is symmetric in p <-> q (Eq.(7)(8)): aggregating a delta
    cost at q seen from p equals the one at p seen from q, up to the
    normalisation; check on unnormalised single-tap responses."""
    rng = np.random.default_rng(15)
    guide = rng.integers(0, 256, (9, 9), dtype=np.uint8)
    wd = oracle_lib.spatial_weights(3, 2.5)
    wr = oracle_lib.range_weights(18.0)
    for _ in range(50):
        p = rng.integers(0, 9, 2); q = p + rng.integers(-3, 4, 2)
        if not (0 <= q[0] < 9 and 0 <= q[1] < 9):
            continue
        w_pq = wd[q[0] - p[0] + 3, q[1] - p[1] + 3] * wr[abs(int(guide[tuple(q)]) - int(guide[tuple(p)]))]
        w_qp = wd[p[0] - q[0] + 3, p[1] - q[1] + 3] * wr[abs(int(guide[tuple(p)]) - int(guide[tuple(q)]))]
        assert w_pq == w_qp
        assert w_pq == pytest.approx(math.exp(-((q[0] - p[0]) ** 2 + (q[1] - p[1]) ** 2) / 2.5 ** 2)
                                     * math.exp(-(int(guide[tuple(q)]) - int(guide[tuple(p)])) ** 2 / 18.0 ** 2),
                                     rel=1e-14)
