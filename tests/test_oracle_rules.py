"""Pins for oracle/rules.py (no GPU).

Each rule is pinned to something other than the oracle itself: the paper's 20-digit
constants, closed forms (P:412 and the symbolic solution of eq:QuadraticQuadrature by
sympy, as Maple did at P:272), exact rational moments from sympy's B-splines,
textbook Gauss-Jacobi rules (scipy) for the boundary classes that reduce to them,
and the paper's wrong Newton root.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import quadrature, rules, spline

PAPER_TOL = 1e-14          # the paper prints 20 digits


@pytest.fixture(scope="module")
def golden(golden_dir):
    with open(os.path.join(golden_dir, "paper_rules.json")) as f:
        return json.load(f)


def _full(tau_half, om_half, L, odd_mid=None):
    """Symmetric completion of a printed half rule on [0, L]."""
    tau = list(tau_half)
    om = list(om_half)
    if odd_mid is not None:
        return np.array(tau + [L - t for t in tau[:-1][::-1]]), np.array(om + om[:-1][::-1])
    return np.array(tau + [L - t for t in tau[::-1]]), np.array(om + om[::-1])


@pytest.mark.parametrize("kind,p", [("mass", 2), ("mass", 3), ("stiffness", 2), ("stiffness", 3)])
def test_interior_rules_match_paper(golden, kind, p):
    g = golden[f"{kind}_p{p}"]
    tau_h = [float(v) for v in g["tau"]]
    om_h = [float(v) for v in g["omega"]]
    if p == 2:     # 3 nodes, the middle one printed last
        tau = np.array([tau_h[0], tau_h[1], 3.0 - tau_h[0]])
        om = np.array([om_h[0], om_h[1], om_h[0]])
    else:
        tau, om = _full(tau_h, om_h, 4.0)
    r = rules.class_rules(p)[kind]["interior"]
    assert np.max(np.abs(r.tau - tau)) < PAPER_TOL
    assert np.max(np.abs(r.omega - om)) < PAPER_TOL
    assert r.residual < 1e-15


def test_p2_mass_matches_symbolic_solution():
    """eq:QuadraticQuadrature as printed, solved symbolically."""
    import sympy as sp
    t1, w1, w2 = sp.symbols("t1 w1 w2", positive=True)
    eqs = [sp.Rational(1, 4) * w1 * t1 ** 2 * (1 - t1) ** 2 - sp.Rational(1, 120),
           sp.Rational(1, 4) * w1 * t1 ** 2 * (-2 * t1 ** 2 + 2 * t1 + 1) + sp.Rational(3, 32) * w2 - sp.Rational(13, 60),
           sp.Rational(1, 2) * w1 * t1 ** 4 + sp.Rational(9, 16) * w2 - sp.Rational(11, 20)]
    sols = [s for s in sp.solve(eqs, [t1, w1, w2], dict=True) if 0 < float(s[t1]) < 1]
    assert len(sols) == 1
    r = rules.class_rules(2)["mass"]["interior"]
    assert abs(r.tau[0] - float(sols[0][t1])) < 1e-15
    assert abs(r.omega[0] - float(sols[0][w1])) < 1e-15
    assert abs(r.omega[1] - float(sols[0][w2])) < 1e-15
    assert abs(float(sols[0][t1]) - (24 - math.sqrt(30)) / 26) < 1e-15


def test_p3_stiffness_tau1_closed_form():
    """eq:CubicStiffTau1: tau1 = 1/2 - sqrt(225 - 30 sqrt 30)/30, quartic residual."""
    r = rules.class_rules(3)["stiffness"]["interior"]
    t1 = 0.5 - math.sqrt(225 - 30 * math.sqrt(30)) / 30
    assert abs(r.tau[0] - t1) < 1e-15
    x = r.tau[0]
    assert abs(30 * x ** 4 - 60 * x ** 3 + 30 * x ** 2 - 1) < 1e-12
    assert rules.cubic_stiff_tau1(1.0)[1] == pytest.approx(0.5 + math.sqrt(225 - 30 * math.sqrt(30)) / 30, abs=1e-14)


@pytest.mark.parametrize("omega1", [0.9, 1.1, 2.0])
def test_p3_stiffness_family(omega1):
    """One-parameter family: other omega1 complete to exact rules (reading R8)."""
    r = rules.interior_stiff_p3(omega1)
    assert r.residual < 1e-13
    with pytest.raises(ValueError):
        rules.cubic_stiff_tau1(0.5)     # real root in (0,1) iff omega1 >= 8/15


def _printed_cubic_mass_system(t1, t2, w1, w2):
    """eq:CubicQuadrature exactly as printed, fixed polynomial pieces."""
    P = t2 ** 3 - 4 * t2 ** 2 + 4 * t2 - 4.0 / 3.0
    return np.array([
        w1 * t1 ** 3 * (1 - t1) ** 3 / 36 - 1 / 5040,
        w1 * t1 ** 3 * (t1 ** 3 / 12 - t1 ** 2 / 6 + 1.0 / 9) - w2 * (2 - t2) ** 3 * P / 12 - 1 / 42,
        -w1 * t1 ** 3 * (t1 ** 3 - t1 ** 2 - t1 - 1.0 / 3) / 12 - w2 * (t2 ** 3 - 4.5 * t2 ** 2 + 6 * t2 - 1.5) * P / 3 - 397 / 1680,
        w1 * t1 ** 6 / 18 + w2 * P ** 2 / 2 - 151 / 315])


def test_wrong_root_of_paper(golden):
    """the printed root with tau2 = 2.3038 solves the printed fixed-piece system
    but violates tau2 in [1,2] and is NOT an exact rule for the true piecewise B-splines;
    the oracle's root solves both."""
    g = golden["wrong_root_p3_mass"]
    t1, t2 = (float(v) for v in g["tau"])
    w1, w2 = (float(v) for v in g["omega"])
    assert np.max(np.abs(_printed_cubic_mass_system(t1, t2, w1, w2))) < 1e-13
    wrong = rules.Rule("mass", 3, "interior", [t1, t2, 4 - t2, 4 - t1], [w1, w2, w2, w1], 0.0)
    assert rules.full_residual(wrong) > 1e-2
    r = rules.class_rules(3)["mass"]["interior"]
    assert np.max(np.abs(_printed_cubic_mass_system(r.tau[0], r.tau[1], r.omega[0], r.omega[1]))) < 1e-15


def _sympy_residual(rule, p, n_ref=None):
    """Full exactness residual with sympy's exact B-splines and exact moments."""
    import sympy as sp
    n_ref = n_ref or 4 * p + 2
    knots = [0] * (p + 1) + list(range(1, n_ref)) + [n_ref] * (p + 1)
    x = sp.Symbol("x")
    B = sp.bspline_basis_set(p, [sp.Rational(k) for k in knots], x)
    j = 2 * p if rule.cls == "interior" else rule.cls[1]
    lo = j - p if rule.cls == "interior" else 0
    hi = j + 1
    order = 0 if rule.kind == "mass" else 1
    F = [sp.diff(b, x, order) if order else b for b in B]
    worst = 0.0
    for i in range(max(0, j - p), j + p + 1):
        exact = float(sp.integrate(sp.piecewise_fold(F[i] * F[j]), (x, lo, hi)))
        fi = sp.lambdify(x, F[i], "math")
        fj = sp.lambdify(x, F[j], "math")
        q = sum(float(w) * float(fi(lo + t)) * float(fj(lo + t)) for t, w in zip(rule.tau, rule.omega))
        worst = max(worst, abs(q - exact))
    return worst


@pytest.mark.parametrize("p", [2, 3])
def test_every_class_exact_against_sympy(p):
    """P4 / north_star: residual < 1e-13 on the full interacting set, every class."""
    cr = rules.class_rules(p)
    for kind in ("mass", "stiffness"):
        for key, rule in cr[kind].items():
            assert rule.residual < 1e-13, (kind, key)
            assert _sympy_residual(rule, p) < 1e-13, (kind, key)


def test_boundary_textbook_special_cases():
    from scipy.special import roots_jacobi
    # (p=3, j=0, mass): weight (1-x)^3 on [0,1] -> 2-point Gauss-Jacobi(alpha=3, beta=0)
    xi, wi = roots_jacobi(2, 3.0, 0.0)
    x = (1 + xi) / 2
    eff = wi / 2 ** 4
    r = rules.class_rules(3)["mass"][0]
    assert np.allclose(r.tau, np.sort(x), atol=1e-15)
    assert np.allclose(r.omega * (1 - r.tau) ** 3, eff[np.argsort(x)], atol=1e-15)
    # (p=2, j=0, stiffness): weight B_0' = -2(1-x) -> 1-point Gauss-Jacobi(1, 0): node 1/3
    r = rules.class_rules(2)["stiffness"][0]
    assert r.m == 1 and abs(r.tau[0] - 1.0 / 3.0) < 1e-15 and abs(r.omega[0] - 0.75) < 1e-15
    # (p=2, j=0, mass): rational rule tau = (1/10, 1/2), omega = (125/486, 1/2)
    r = rules.class_rules(2)["mass"][0]
    assert np.allclose(r.tau, [0.1, 0.5], atol=1e-15) and np.allclose(r.omega, [125 / 486, 0.5], atol=1e-15)


def test_gl_fallback_classes_have_no_admissible_minimal_rule():
    """Reading R1: stiffness j=1 (p=2, p=3) has no admissible minimal-node rule under the
    midpoint tie-break, so those classes use per-element GL(p+1)."""
    for (kind, p, j) in sorted(rules.GL_FALLBACK):
        rule, count = rules.boundary_gauss(kind, p, j, grid_points=12)
        assert rule is None and count == 0, (kind, p, j)
        g = rules.class_rules(p)[kind][j]
        assert g.m == (p + 1) * (j + 1)


@pytest.mark.slow
def test_boundary_rules_unique():
    """Reading R1 claims a unique admissible root for the other boundary classes."""
    for p in (2, 3):
        for kind in ("mass", "stiffness"):
            for j in range(p):
                if (kind, p, j) in rules.GL_FALLBACK:
                    continue
                rule, count = rules.boundary_gauss(kind, p, j, grid_points=11)
                assert count == 1, (kind, p, j, count)
                assert np.allclose(rule.tau, rules.class_rules(p)[kind][j].tau, atol=1e-12)


@pytest.mark.parametrize("p", [2, 3])
def test_effective_weight_sums(p):
    """P4: sum_k omega_k W(tau_k) = int W (the constant function is in each exactness class)."""
    cr = rules.class_rules(p)
    t, _ = rules.reference_knots(p)
    for kind in ("mass", "stiffness"):
        order = 0 if kind == "mass" else 1
        for key, rule in cr[kind].items():
            j = rules.interior_index(p) if key == "interior" else key
            lo, hi = spline.support(t, j, p)
            W = spline.deriv(t, j, p, lo + rule.tau, order)
            s = float(np.sum(rule.omega * W))
            if kind == "mass":
                expect = 1.0 if key == "interior" else (j + 1) / (p + 1)
            else:
                expect = float(spline.basis(t, j, p, np.array([hi]))[0] - spline.basis(t, j, p, np.array([lo]))[0]) \
                    if key != "interior" else 0.0
                if key == 0:
                    expect = -1.0
            assert abs(s - expect) < 1e-14, (kind, key, s, expect)


@pytest.mark.parametrize("p,n", [(2, 2), (2, 5), (3, 3), (3, 4), (3, 11)])
@pytest.mark.parametrize("mode", ["gauss", "gl"])
def test_mesh_rules_exact_every_row(p, n, mode):
    """Scaling covariance + mirroring: on the physical mesh (h = 1/n) every row's rule
    reproduces int F_i W_r (F = B or B') for all interacting i, including right-boundary
    mirrored classes and n = p (the smallest admissible mesh)."""
    t = spline.open_uniform_knots(p, n)
    N = n + p
    for kind in ("mass", "stiffness"):
        order = 0 if kind == "mass" else 1
        R = rules.rules_1d(p, n, kind, mode)
        for r in range(N):
            lo, hi = spline.support(t, r, p)
            assert np.all(R[r].x > lo) and np.all(R[r].x < hi)
            for i in spline.interacting(p, n, r):
                exact = quadrature.product_integral(t, p, i, r, order, order, lo, hi)
                q = float(np.sum(R[r].w * spline.deriv(t, i, p, R[r].x, order)))
                assert abs(q - exact) < 1e-13 * max(1.0, n ** (2 * order - 1)), (kind, r, i, q, exact)


def test_unsupported():
    with pytest.raises(ValueError):
        rules.rules_1d(3, 2, "mass")
    with pytest.raises(ValueError):
        rules.class_rules(4)
    assert list(itertools.islice(rules.GL_FALLBACK, 0))  == []
