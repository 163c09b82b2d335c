"""Pins for oracle/spline.py and oracle/quadrature.py (no GPU).

The oracle's Cox-de Boor basis is checked against an independent library routine
(scipy.interpolate.BSpline), against the SPEC example values and against the
partition-of-unity identities; Gauss-Legendre against monomial integrals; the exact
moments against the paper's printed right-hand sides and against sympy's exact
piecewise-polynomial B-splines.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy.interpolate import BSpline

from oracle import quadrature, spline


@pytest.mark.parametrize("p", [2, 3])
@pytest.mark.parametrize("n", [1, 3, 4, 7, 16])
def test_basis_matches_scipy(p, n):
    if n < 1:
        return
    t = spline.open_uniform_knots(p, n)
    rng = np.random.default_rng(100 * p + n)
    x = np.concatenate([rng.uniform(0, 1, 200), t[p:-p], [0.0, 1.0]])
    x = np.clip(x, 0.0, 1.0)
    N = spline.dim(p, n)
    for i in range(N):
        c = np.zeros(N)
        c[i] = 1.0
        ref = BSpline(t, c, p, extrapolate=False)
        mine = spline.basis(t, i, p, x)
        assert np.allclose(mine, np.nan_to_num(ref(x)), atol=1e-14, rtol=0), (p, n, i)
        # derivatives away from knots (derivatives of C^{p-1} splines are continuous for p >= 2)
        xi = rng.uniform(0, 1, 100)
        for order in (1, 2):
            dref = ref.derivative(order)(xi)
            dmine = spline.deriv(t, i, p, xi, order)
            assert np.allclose(dmine, dref, atol=1e-10 * n ** order, rtol=1e-12), (p, n, i, order)


def test_spec_examples():
    # cardinal centre functions: p=2 B(1.5)=3/4, p=3 B(2)=2/3, p=2 B'(0.75)=0.75, B'(1.5)=0
    t2 = spline.open_uniform_knots(2, 10, length=10.0)   # unit spacing
    j2 = 4                                                # supp [2, 5], cardinal
    assert spline.basis(t2, j2, 2, np.array([2 + 1.5]))[0] == pytest.approx(0.75, abs=1e-15)
    assert spline.deriv(t2, j2, 2, np.array([2 + 0.75]), 1)[0] == pytest.approx(0.75, abs=1e-15)
    assert abs(spline.deriv(t2, j2, 2, np.array([2 + 1.5]), 1)[0]) < 1e-15
    t3 = spline.open_uniform_knots(3, 12, length=12.0)
    j3 = 6                                                # supp [3, 7]
    assert spline.basis(t3, j3, 3, np.array([3 + 2.0]))[0] == pytest.approx(2.0 / 3.0, abs=1e-15)
    assert abs(spline.deriv(t3, j3, 3, np.array([3 + 2.0]), 1)[0]) < 1e-15
    # endpoint interpolation of open knots, dim = p + n (eq:DimUni)
    t = spline.open_uniform_knots(3, 5)
    assert spline.basis(t, 0, 3, np.array([0.0]))[0] == 1.0
    assert spline.basis(t, 7, 3, np.array([1.0]))[0] == 1.0
    assert spline.dim(3, 5) == len(t) - 3 - 1 == 8


@pytest.mark.parametrize("p", [2, 3])
def test_partition_of_unity(p):
    n = 9
    t = spline.open_uniform_knots(p, n)
    x = np.random.default_rng(p).uniform(0, 1, 1000)
    S = sum(spline.basis(t, i, p, x) for i in range(spline.dim(p, n)))
    dS = sum(spline.deriv(t, i, p, x, 1) for i in range(spline.dim(p, n)))
    assert np.max(np.abs(S - 1)) < 1e-13
    assert np.max(np.abs(dS)) < 1e-11
    assert min(np.min(spline.basis(t, i, p, x)) for i in range(spline.dim(p, n))) > -1e-15


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6])
def test_gauss_legendre_exact_on_monomials(m):
    x, w = quadrature.gauss_legendre(m, 0.0, 1.0)
    for k in range(2 * m):
        assert abs(np.sum(w * x ** k) - 1.0 / (k + 1)) < 1e-15
    x, w = quadrature.gauss_legendre(m, 2.0, 5.0)
    assert abs(np.sum(w * x ** (2 * m - 1)) - (5.0 ** (2 * m) - 2.0 ** (2 * m)) / (2 * m)) < 1e-10 * 5.0 ** (2 * m)


def _golden(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("kind,p", [("mass", 2), ("mass", 3), ("stiffness", 2), ("stiffness", 3)])
def test_interior_moments_match_paper(golden_dir, kind, p):
    g = _golden(golden_dir, "paper_moments.json")[f"{kind}_p{p}"]
    sign = g.get("sign", [1] * len(g["num"]))
    expect = [s * a / b for s, a, b in zip(sign, g["num"], g["den"])]
    t = spline.open_uniform_knots(p, 4 * p + 2, length=4 * p + 2.0)
    j = 2 * p
    mine = quadrature.moments(t, p, j, kind, list(range(j - p, j + 1)))
    assert np.allclose(mine, expect, atol=1e-15, rtol=1e-14)


def _sympy_basis(p, knots):
    import sympy as sp
    x = sp.Symbol("x")
    return x, sp.bspline_basis_set(p, [sp.Rational(k) for k in knots], x)


@pytest.mark.parametrize("p", [2, 3])
def test_all_moments_match_sympy_exact(p):
    """Every exactness right-hand side (interior and boundary classes, mass and
    stiffness) against exact rational integration of sympy's B-splines."""
    import sympy as sp
    n_ref = 4 * p + 2
    knots = [0] * (p + 1) + list(range(1, n_ref)) + [n_ref] * (p + 1)
    x, B = _sympy_basis(p, knots)
    t = spline.open_uniform_knots(p, n_ref, length=float(n_ref))
    for j in list(range(p)) + [2 * p]:
        lo, hi = (0, j + 1) if j < p else (j - p, j + 1)
        rows = [i for i in range(j - p, j + p + 1) if i >= 0]
        for kind in ("mass", "stiffness"):
            mine = quadrature.moments(t, p, j, kind, rows)
            for i, v in zip(rows, mine):
                fi, fj = (B[i], B[j]) if kind == "mass" else (sp.diff(B[i], x), sp.diff(B[j], x))
                exact = sp.integrate(sp.piecewise_fold(fi * fj), (x, lo, hi))
                assert abs(v - float(exact)) < 1e-15, (p, j, kind, i, v, exact)


def test_moment_fraction_examples():
    # Appendix B of SURVEY.md spot values, cross-checked here with fractions:
    # p=2 left boundary row 0: int B_0^2 = 1/5 (B_0 = (1-x)^2 on [0,1])
    t = spline.open_uniform_knots(2, 10, length=10.0)
    assert abs(quadrature.product_integral(t, 2, 0, 0) - float(Fraction(1, 5))) < 4e-16
    # stiffness: int (B_0')^2 = int 4(1-x)^2 = 4/3
    assert abs(quadrature.product_integral(t, 2, 0, 0, 1, 1) - 4.0 / 3.0) < 1e-15
