"""Gauss-Legendre and exact spline moments -- ORACLE (test infrastructure only).

The right-hand sides of the exactness systems eq:GaussQuadSys and
eq:GaussQuadSysStiff are integrals of products of two degree-p
(resp. p-1) piecewise polynomials with breakpoints at the knots.  On each knot
span the product is a polynomial of degree <= 2p, which m-point Gauss-Legendre
integrates exactly for 2m-1 >= 2p; we use m = p + 2 (one spare degree).

Gauss-Legendre nodes/weights come from the library routine numpy's ``leggauss``
(pinned in tests against monomial integrals).
"""
import numpy as np

from . import spline


def gauss_legendre(m, a=0.0, b=1.0):
    """m-point Gauss-Legendre rule on [a, b]."""
    x, w = np.polynomial.legendre.leggauss(m)
    return 0.5 * (b - a) * x + 0.5 * (a + b), 0.5 * (b - a) * w


def spans(t, lo, hi):
    """Non-empty knot spans [t_s, t_{s+1}] inside [lo, hi]."""
    out = []
    for s in range(len(t) - 1):
        a, b = float(t[s]), float(t[s + 1])
        if b > a and a >= lo and b <= hi:
            out.append((a, b))
    return out


def product_integral(t, k, i, j, di=0, dj=0, lo=None, hi=None, m=None):
    """int_{lo}^{hi} B_i^{(di)} B_j^{(dj)} dx, exact by per-span Gauss-Legendre."""
    if lo is None:
        lo = float(t[0])
    if hi is None:
        hi = float(t[-1])
    if m is None:
        m = k + 2
    total = 0.0
    for a, b in spans(t, lo, hi):
        x, w = gauss_legendre(m, a, b)
        total += float(np.sum(w * spline.deriv(t, i, k, x, di) * spline.deriv(t, j, k, x, dj)))
    return total


def moments(t, k, j, kind, rows):
    """Exactness right-hand sides for the weight B_j (mass) or B'_j (stiffness).

    mass:      mu_i = int_{supp B_j} B_i B_j        (eq:GaussQuadSys)
    stiffness: mu_i = int_{supp B_j} B'_i B'_j      (eq:GaussQuadSysStiff)
    for every i in ``rows`` (the functions interacting with B_j).
    Signs are the true ones (reading R3; the paper prints magnitudes).
    """
    lo, hi = spline.support(t, j, k)
    d = 0 if kind == "mass" else 1
    return np.array([product_integral(t, k, i, j, d, d, lo, hi) for i in rows])
