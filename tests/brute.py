"""Literal brute force of the FBS definitions, for tiny inputs only.

Written independently of oracle/fbs_oracle.c to pin it: no precomputed block
statistics, no twin write, no weight tables, two-pass (covariance) statistics
instead of the one-pass Eq.(2)(3) form, ``math.exp`` per tap.  Pure Python
loops; do not call on anything larger than ~16x16x8.
"""
from __future__ import annotations

import math
from decimal import Decimal, getcontext

SENT = -2.0


def _block(img, u, v):
    return [int(img[y][x]) for y in (v - 1, v, v + 1) for x in (u - 1, u, u + 1)]


def ncc(L, R, u, v, d):
    """Eq.(1) as a Pearson correlation of the two 3x3 blocks (covariance form)."""
    H, W = len(L), len(L[0])
    if not (1 <= u <= W - 2 and 1 <= v <= H - 2 and 1 <= u - d <= W - 2):
        return SENT
    a = _block(L, u, v)
    b = _block(R, u - d, v)
    ma = sum(a) / 9.0
    mb = sum(b) / 9.0
    sa = math.sqrt(sum((x - ma) ** 2 for x in a) / 9.0)
    sb = math.sqrt(sum((x - mb) ** 2 for x in b) / 9.0)
    if sa < 1e-6 or sb < 1e-6:
        return SENT
    c = sum((x - ma) * (y - mb) for x, y in zip(a, b)) / (9.0 * sa * sb)
    return max(-1.0, min(1.0, c))


def ncc_exact(L, R, u, v, d, digits: int = 50):
    """Eq.(1) in exact integer arithmetic, rounded once: N / sqrt(V_l V_r) with
    N = 9 Σ a b − S_a S_b and V = 9 Σ a^2 − S^2 (algebraically identical to
    Eq.(1)-(3)), evaluated with ``digits`` significant decimal digits."""
    H, W = len(L), len(L[0])
    if not (1 <= u <= W - 2 and 1 <= v <= H - 2 and 1 <= u - d <= W - 2):
        return SENT
    a = _block(L, u, v)
    b = _block(R, u - d, v)
    Sa, Sb = sum(a), sum(b)
    Va = 9 * sum(x * x for x in a) - Sa * Sa
    Vb = 9 * sum(x * x for x in b) - Sb * Sb
    if Va == 0 or Vb == 0:
        return SENT
    N = 9 * sum(x * y for x, y in zip(a, b)) - Sa * Sb
    getcontext().prec = digits
    c = Decimal(N) / (Decimal(Va) * Decimal(Vb)).sqrt()
    return float(max(Decimal(-1), min(Decimal(1), c)))


def cost_volumes(L, R, d_min, d_max):
    """Left and right volumes [v][u][d-d_min]; the right one is evaluated in its
    own frame (right block at x', left block at x'+d), not copied."""
    H, W = len(L), len(L[0])
    D = d_max - d_min + 1
    cl = [[[ncc(L, R, u, v, d_min + k) for k in range(D)] for u in range(W)] for v in range(H)]
    cr = [[[ncc(L, R, u + d_min + k, v, d_min + k) if u + d_min + k < W else SENT for k in range(D)]
           for u in range(W)] for v in range(H)]
    return cl, cr


def aggregate(cost, guide, rho, gamma_d, gamma_r):
    """Eq.(6)-(8) literally: exp() per tap, window truncated, SENT taps skipped."""
    H, W, D = len(cost), len(cost[0]), len(cost[0][0])
    out = [[[SENT] * D for _ in range(W)] for _ in range(H)]
    for v in range(H):
        for u in range(W):
            for k in range(D):
                num = den = 0.0
                any_ = False
                for y in range(v - rho, v + rho + 1):
                    for x in range(u - rho, u + rho + 1):
                        if not (0 <= x < W and 0 <= y < H):
                            continue
                        c = cost[y][x][k]
                        if c == SENT:
                            continue
                        wd = math.exp(-((x - u) ** 2 + (y - v) ** 2) / gamma_d ** 2)
                        wr = math.exp(-((int(guide[y][x]) - int(guide[v][u])) ** 2) / gamma_r ** 2)
                        num += wd * wr * c
                        den += wd * wr
                        any_ = True
                if any_:
                    out[v][u][k] = num / den
    return out


def wta(col, d_min):
    """argmax over defined entries, smallest d on ties; None if all SENT."""
    defined = [(c, k) for k, c in enumerate(col) if c != SENT]
    if not defined:
        return None
    best = max(c for c, _ in defined)
    return d_min + min(k for c, k in defined if c == best)


def subpixel(cm, c0, cp, d):
    den = 2 * cm + 2 * cp - 4 * c0
    if abs(den) < 1e-9:
        return float(d)
    return d + max(-0.5, min(0.5, (cm - cp) / den))


def pipeline(L, R, d_min, d_max, rho, gamma_d, gamma_r):
    """Whole method; returns the subpixel map as nested lists (-1.0 invalid)."""
    H, W = len(L), len(L[0])
    D = d_max - d_min + 1
    cl, cr = cost_volumes(L, R, d_min, d_max)
    al = aggregate(cl, L, rho, gamma_d, gamma_r)
    ar = aggregate(cr, R, rho, gamma_d, gamma_r)
    dl = [[wta(al[v][u], d_min) for u in range(W)] for v in range(H)]
    dr = [[wta(ar[v][u], d_min) for u in range(W)] for v in range(H)]
    out = [[-1.0] * W for _ in range(H)]
    for v in range(H):
        for u in range(W):
            d = dl[v][u]
            if d is None or u - d < 0 or dr[v][u - d] is None or abs(d - dr[v][u - d]) > 1:
                continue
            k = d - d_min
            if 0 < k < D - 1 and al[v][u][k - 1] != SENT and al[v][u][k + 1] != SENT:
                out[v][u] = subpixel(al[v][u][k - 1], al[v][u][k], al[v][u][k + 1], d)
            else:
                out[v][u] = float(d)
    return out, dl, dr, al, ar
