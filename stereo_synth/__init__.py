"""Seeded synthetic stereo pairs shared by the oracle tests, the GPU parity tests
and bench.py.

This module holds NO arithmetic of the FBS method (no NCC, no weights, no
aggregation): it only makes uint8 image pairs.  Both the oracle side and the
CUDA side consume the same bytes.  The draw order is part of the contract and
versioned by ``SYNTH_VERSION``; DESIGN.md §5 states the recipe.

Workload shapes follow BASELINE.json ``configs`` (Middlebury 2001/2003-like
scenes: "Middlebury 2001 datasets and 2003 datasets").
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

SYNTH_VERSION = 1


@dataclass(frozen=True)
class Config:
    name: str
    W: int
    H: int
    d_min: int
    d_max: int
    radius: int
    seed: int
    gamma_d: float = 5.0   # sigma_s (γ_d of Eq.(7)); unstated in the paper (R#27)
    gamma_r: float = 32.0  # sigma_r (γ_r of Eq.(8)); >= 27.3 avoids fp32 underflow (R#13)

    @property
    def D(self) -> int:
        return self.d_max - self.d_min + 1


# BASELINE.json configs[0..4]
CONFIGS = {
    "synthetic": Config("synthetic", 64, 48, 0, 15, 3, 0x1807),
    "tsukuba": Config("tsukuba", 384, 288, 0, 15, 4, 0x1808),
    "teddy": Config("teddy", 450, 375, 0, 59, 4, 0x1809),
    "mb2014": Config("mb2014", 2880, 1988, 0, 255, 4, 0x180A),
    "kitti": Config("kitti", 1242, 375, 0, 127, 4, 0x2000),
}


def random_dot(W: int, H: int, shift: int, seed: int):
    """I_L ~ U{0..255} i.i.d.; I_R(x, y) = I_L(x + s, y), fresh U{0..255} where
    x + s >= W.  Returns (left, right) uint8 [H, W]."""
    rng = np.random.default_rng(seed)
    left = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    fresh = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    right = fresh.copy()
    if shift < W:
        right[:, : W - shift] = left[:, shift:]
    return left, right


def _layer_texture(rng, W: int, H: int, p_flat: float = 0.1) -> np.ndarray:
    """One layer's 8-bit texture over the whole frame (draw order fixed)."""
    if rng.random() < p_flat:  # textureless layer -> V = 0 blocks -> undefined costs
        return np.full((H, W), int(rng.integers(30, 226)), dtype=np.uint8)
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    t = np.full((H, W), 128.0)
    for _ in range(3):
        f = rng.uniform(0.02, 0.25)
        th = rng.uniform(0.0, 2 * np.pi)
        ph = rng.uniform(0.0, 2 * np.pi)
        t += 20.0 * np.sin(2 * np.pi * f * (xx * np.cos(th) + yy * np.sin(th)) + ph)
    t += rng.normal(0.0, 6.0, size=(H, W))
    return np.clip(np.rint(t), 0, 255).astype(np.uint8)


def layered(W: int, H: int, d_min: int, d_max: int, seed: int, n_rects: int = 6,
            photometric: bool = True, p_flat: float = 0.1):
    """Middlebury-like layered scene: a background plane plus ``n_rects``
    fronto-parallel textured rectangles at integer disparities.

    Returns (left, right, gt_disp int32 [H,W], occluded bool [H,W]).  The ground
    truth is for logging only (PEP is out of scope)."""
    rng = np.random.default_rng(seed)
    D = d_max - d_min + 1
    disp = np.full((H, W), d_min + D // 8, dtype=np.int32)
    left = _layer_texture(rng, W, H, p_flat)
    for _ in range(n_rects):
        rw = int(rng.integers(max(1, W // 8), max(2, W // 3) + 1))
        rh = int(rng.integers(max(1, H // 8), max(2, H // 3) + 1))
        cx = int(rng.integers(0, W)); cy = int(rng.integers(0, H))
        dd = int(rng.integers(d_min + D // 4, max(d_min + D // 4 + 1, d_max)))
        tex = _layer_texture(rng, W, H, p_flat)
        x0, x1 = max(0, cx - rw // 2), min(W, cx - rw // 2 + rw)
        y0, y1 = max(0, cy - rh // 2), min(H, cy - rh // 2 + rh)
        left[y0:y1, x0:x1] = tex[y0:y1, x0:x1]
        disp[y0:y1, x0:x1] = dd
    fresh = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    right = fresh.copy()
    ys, xs = np.mgrid[0:H, 0:W]
    # forward warp I_R(x - d, y) = I_L(x, y); z-buffer: larger d wins (ascending levels)
    for d in np.unique(disp):
        m = (disp == d) & (xs - d >= 0)
        right[ys[m], xs[m] - d] = left[m]
    # a left pixel is occluded if its right target was overwritten by a nearer layer
    occl = np.ones((H, W), dtype=bool)
    xr = xs - disp
    ok = xr >= 0
    winner = np.full((H, W), -1, dtype=np.int32)
    for d in np.unique(disp):
        m = (disp == d) & ok
        winner[ys[m], xr[m]] = d
    occl[ok] = winner[ys[ok], xr[ok]] != disp[ok]
    if photometric:  # gain/offset change: NCC is invariant to it
        right = np.clip(np.rint(0.9 * right.astype(np.float64) + 10.0), 0, 255).astype(np.uint8)
    return left, right, disp, occl


def frame(cfg: Config, index: int = 0, kind: str = "layered"):
    """The (left, right) pair of frame ``index`` for a config (seed + index)."""
    seed = cfg.seed + index
    if kind == "layered":
        left, right, _, _ = layered(cfg.W, cfg.H, cfg.d_min, cfg.d_max, seed)
    elif kind == "random_dot":
        shift = cfg.d_min + (seed % cfg.D)
        left, right = random_dot(cfg.W, cfg.H, shift, seed)
    else:
        raise ValueError(kind)
    return left, right


def digest(*arrays) -> str:
    """SHA-256 of the input bytes (logged beside every result)."""
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
