"""1D numerics restated from the reference (TEST INFRASTRUCTURE ONLY).

Each function cites the reference routine whose behaviour it restates:

* legendre            quadrature.py:57-75
* jacobi / jacobi_deriv quadrature.py:78-102
* gll / gl / radau    quadrature.py:153-185 (bracketing + Newton there;
                      here Newton from Chebyshev guesses in extended
                      precision — same roots to < 1e-15)
* diff_matrix         quadrature.py:224-260 (barycentric form)
* modified_a          basis.py:78-96 + boundary_first_permutation basis.py:111-114
                      (storage order of stdregions.py:56-67)
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

GLL = "gauss_lobatto_legendre"
GL = "gauss_legendre"
RADAU_M = "gauss_radau_m_legendre"


def legendre(n, x):
    """P_n(x) and P_n'(x) by the three-term recurrence (quadrature.py:57-75)."""
    x = np.asarray(x, dtype=np.longdouble)
    p0 = np.ones_like(x)
    if n == 0:
        return p0, np.zeros_like(x)
    p1 = x.copy()
    for k in range(1, n):
        p0, p1 = p1, ((2 * k + 1) * x * p1 - k * p0) / (k + 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        dp = n * (p0 - x * p1) / (1 - x * x)
    end = np.abs(np.abs(x) - 1) < 1e-30
    if np.any(end):
        sgn = np.where(x > 0, 1.0, (-1.0) ** (n - 1))
        dp = np.where(end, sgn * n * (n + 1) / 2.0, dp)
    return p1, dp


def jacobi(n, a, b, x):
    """P_n^{a,b}(x), three-term recurrence (quadrature.py:78-95)."""
    x = np.asarray(x, dtype=float)
    p0 = np.ones_like(x)
    if n == 0:
        return p0
    p1 = 0.5 * ((a + b + 2) * x + (a - b))
    for k in range(2, n + 1):
        c = 2 * k + a + b
        a1 = 2 * k * (k + a + b) * (c - 2)
        a2 = (c - 1) * (a * a - b * b)
        a3 = (c - 2) * (c - 1) * c
        a4 = 2 * (k + a - 1) * (k + b - 1) * c
        p0, p1 = p1, ((a2 + a3 * x) * p1 - a4 * p0) / a1
    return p1


def jacobi_deriv(n, a, b, x):
    """d/dx P_n^{a,b} (quadrature.py:98-102)."""
    if n == 0:
        return np.zeros_like(np.asarray(x, dtype=float))
    return 0.5 * (n + a + b + 1) * jacobi(n - 1, a + 1, b + 1, x)


def _newton(f_df, x0, iters=60):
    x = np.asarray(x0, dtype=np.longdouble)
    for _ in range(iters):
        f, df = f_df(x)
        step = f / df
        x = x - step
        if np.max(np.abs(step)) < 1e-19:
            break
    return x


@lru_cache(maxsize=None)
def rule(q: int, ptype: str = GLL):
    """(points, weights) of a Q-point rule on [-1,1] (quadrature.py:188-214)."""
    if ptype == GLL:
        if q < 2:
            raise ValueError("Gauss-Lobatto-Legendre needs at least 2 points")
        if q == 2:
            return np.array([-1.0, 1.0]), np.array([1.0, 1.0])
        n = q - 1
        # interior nodes: roots of P_n' (quadrature.py:153-166)
        x0 = -np.cos(np.pi * np.arange(1, q - 1) / n)

        def f_df(x):
            p, dp = legendre(n, x)
            d2p = (2 * x * dp - n * (n + 1) * p) / (1 - x * x)
            return dp, d2p

        xi = _newton(f_df, x0)
        pts = np.concatenate(([-1.0], np.asarray(xi, float), [1.0]))
        p, _ = legendre(n, np.concatenate(([-1.0], xi, [1.0])).astype(np.longdouble))
        wts = np.asarray(2.0 / (q * n * p * p), float)
    elif ptype == GL:
        if q == 1:
            return np.array([0.0]), np.array([2.0])
        x0 = -np.cos(np.pi * (np.arange(q) + 0.75) / (q + 0.5))
        xi = _newton(lambda x: legendre(q, x), x0)
        _, dp = legendre(q, xi)
        pts = np.asarray(xi, float)
        wts = np.asarray(2.0 / ((1 - xi * xi) * dp * dp), float)
    elif ptype == RADAU_M:
        if q == 1:
            return np.array([-1.0]), np.array([2.0])
        n = q - 1
        # interior: roots of P_n^{(0,1)} (quadrature.py:169-185); their
        # Newton guesses come from the Radau nodes of Chebyshev type.
        x0 = -np.cos(2 * np.pi * np.arange(1, q) / (2 * q - 1))

        def f_df(x):
            xf = x.astype(float)
            return (np.asarray(jacobi(n, 0.0, 1.0, xf), np.longdouble),
                    np.asarray(jacobi_deriv(n, 0.0, 1.0, xf), np.longdouble))

        xi = _newton(f_df, x0)
        xi = np.asarray(xi, float)
        pts = np.concatenate(([-1.0], xi))
        p, _ = legendre(n, xi)
        wts = np.empty(q)
        wts[0] = 2.0 / (q * q)
        wts[1:] = np.asarray((1.0 - xi) / (q * q * p * p), float)
    else:
        raise ValueError(f"unknown points type {ptype}")
    pts = np.asarray(pts, float)
    wts = np.asarray(wts, float)
    pts.setflags(write=False)
    wts.setflags(write=False)
    return pts, wts


def diff_matrix(points):
    """Collocation derivative matrix, barycentric form (quadrature.py:246-260)."""
    x = np.asarray(points, dtype=float)
    q = len(x)
    diff = x[:, None] - x[None, :]
    np.fill_diagonal(diff, 1.0)
    bw = 1.0 / diff.prod(axis=1)
    d = np.zeros((q, q))
    for i in range(q):
        for j in range(q):
            if i != j:
                d[i, j] = (bw[j] / bw[i]) / (x[i] - x[j])
        d[i, i] = -d[i].sum()
    return d


def modified_a(P, points):
    """Modified_A values/derivatives in boundary-first storage order.

    basis.py:78-96 (formula order) permuted by basis.py:111-114:
    row 0 = (1-x)/2, row 1 = (1+x)/2, row k>=2 = lo*hi*P^{1,1}_{k-2}(x).
    """
    z = np.asarray(points, dtype=float)
    lo, hi = 0.5 * (1 - z), 0.5 * (1 + z)
    vals = [lo, hi]
    ders = [np.full_like(z, -0.5), np.full_like(z, 0.5)]
    for k in range(2, P + 1):
        j = jacobi(k - 2, 1.0, 1.0, z)
        dj = jacobi_deriv(k - 2, 1.0, 1.0, z)
        vals.append(lo * hi * j)
        ders.append(-0.5 * z * j + lo * hi * dj)
    return np.array(vals), np.array(ders)


class Tables1D:
    """Everything one direction needs: m modes, Q points of one type."""

    def __init__(self, m: int, q: int, ptype: str = GLL):
        self.m, self.q, self.ptype = m, q, ptype
        self.z, self.w = rule(q, ptype)
        self.B, self.Bd = modified_a(m - 1, self.z)     # (m, Q)
        self.D = diff_matrix(self.z)                    # (Q, Q)


@lru_cache(maxsize=None)
def tables(m: int, q: int, ptype: str = GLL) -> Tables1D:
    return Tables1D(m, q, ptype)
