"""A second, independent numpy implementation of hdiff and vadv.  TEST INFRASTRUCTURE ONLY.

Written from the same definitions as oracle/oec_oracle.c (readings R1-R11) but with
whole-array slicing instead of point loops, so a slip in either (an index, a sign, an operand
order) shows up as a mismatch.  numpy elementwise fp64 arithmetic is IEEE RNE without
contraction, so the two agree bitwise.  float32 fields give the binary32 instance:
numpy keeps float32 arithmetic in float32 and rounds Python-float constants to float32 (NEP 50),
as the C oracle's R() does.
"""
from __future__ import annotations

import numpy as np

from synth import HostField


def _sl(f: HostField, i0, i1, j0, j1, k0, k1):
    return f.data[k0 - f.lb[2]:k1 - f.lb[2], j0 - f.lb[1]:j1 - f.lb[1], i0 - f.lb[0]:i1 - f.lb[0]]


def hdiff(inp: HostField, coeff: HostField, lo, hi, limiter: bool = True) -> np.ndarray:
    """Returns out over the domain [lo, hi) as an array [k][j][i]."""
    (i0, j0, k0), (i1, j1, k1) = lo, hi

    def IN(di, dj, a0, a1, b0, b1):  # in over i in [a0,a1), j in [b0,b1), shifted
        return _sl(inp, a0 + di, a1 + di, b0 + dj, b1 + dj, k0, k1)

    # lap on [i0-1, i1+1) x [j0-1, j1+1)
    L = (i0 - 1, i1 + 1, j0 - 1, j1 + 1)
    lap = ((IN(-1, 0, *L) + IN(1, 0, *L)) + (IN(0, -1, *L) + IN(0, 1, *L))) - 4.0 * IN(0, 0, *L)

    def LAP(di, dj, a0, a1, b0, b1):
        return lap[:, b0 + dj - (j0 - 1):b1 + dj - (j0 - 1), a0 + di - (i0 - 1):a1 + di - (i0 - 1)]

    X = (i0 - 1, i1, j0, j1)
    f = LAP(1, 0, *X) - LAP(0, 0, *X)
    flx = np.where(f * (IN(1, 0, *X) - IN(0, 0, *X)) > 0.0, 0.0, f) if limiter else f
    Y = (i0, i1, j0 - 1, j1)
    g = LAP(0, 1, *Y) - LAP(0, 0, *Y)
    fly = np.where(g * (IN(0, 1, *Y) - IN(0, 0, *Y)) > 0.0, 0.0, g) if limiter else g
    D = (i0, i1, j0, j1)
    c = _sl(coeff, i0, i1, j0, j1, k0, k1)
    return IN(0, 0, *D) - c * ((flx[:, :, 1:] - flx[:, :, :-1]) + (fly[:, 1:, :] - fly[:, :-1, :]))


def vadv(f, dtr: float, lo, hi) -> np.ndarray:
    """Thomas solve per column, vectorised over (j, i); returns utens_stage_out [k][j][i]."""
    (i0, j0, k0), (i1, j1, k1) = lo, hi
    K = k1 - k0
    BET_M = BET_P = 0.5

    def F(name, k, di=0):
        return _sl(f[name], i0 + di, i1 + di, j0, j1, k, k + 1)[0]

    a = [None] * K
    b = [None] * K
    c = [None] * K
    d = [None] * K
    for q in range(K):
        k = k0 + q
        if q == 0:
            gcv = 0.25 * (F("wcon", k + 1, 1) + F("wcon", k + 1))
            a[q] = np.zeros_like(gcv)
            c[q] = gcv * BET_P
            b[q] = dtr - c[q]
            corr = -(gcv * BET_M) * (F("u_stage", k + 1) - F("u_stage", k))
        elif q == K - 1:
            gav = -0.25 * (F("wcon", k, 1) + F("wcon", k))
            a[q] = gav * BET_P
            c[q] = np.zeros_like(gav)
            b[q] = dtr - a[q]
            corr = -(gav * BET_M) * (F("u_stage", k - 1) - F("u_stage", k))
        else:
            gav = -0.25 * (F("wcon", k, 1) + F("wcon", k))
            gcv = 0.25 * (F("wcon", k + 1, 1) + F("wcon", k + 1))
            a[q] = gav * BET_P
            c[q] = gcv * BET_P
            b[q] = (dtr - a[q]) - c[q]
            corr = (-(gav * BET_M) * (F("u_stage", k - 1) - F("u_stage", k))) - (gcv * BET_M) * (
                F("u_stage", k + 1) - F("u_stage", k))
        d[q] = ((dtr * F("u_pos", k) + F("utens", k)) + F("utens_stage_in", k)) + corr
    cp = [None] * K
    dp = [None] * K
    r = 1.0 / b[0]
    cp[0], dp[0] = c[0] * r, d[0] * r
    for q in range(1, K):
        r = 1.0 / (b[q] - cp[q - 1] * a[q])
        cp[q] = c[q] * r
        dp[q] = (d[q] - dp[q - 1] * a[q]) * r
    out = np.empty((K, j1 - j0, i1 - i0), dtype=dp[0].dtype)
    x = dp[K - 1]
    out[K - 1] = dtr * (x - F("u_pos", k0 + K - 1))
    for q in range(K - 2, -1, -1):
        x = dp[q] - cp[q] * x
        out[q] = dtr * (x - F("u_pos", k0 + q))
    return out
