"""Basis-evaluation counts of the row-wise schemes -- ORACLE (test infrastructure only).

SURVEY §8(f) row 3 / experiment E3 (fig:ResultQuadCalls and the remark P:478-481):
the paper's cost metric is "the number of basis function evaluations at the quadrature
points required to build the mass matrix", compared between the weighted Gaussian rules and
the weighted Newton-Cotes rules of Calabro et al., whose points are the knots and element
midpoints, "excluding from our counting the cases where the function
evaluation is redundant".  Counting protocol (SURVEY §6 [V]):

* per 1D row r and node x of its rule: the number of the 2p+1 interacting functions
  B_{r+o} (mass) or B'_{r+o} (stiffness) that are nonzero at x;
* Gaussian: the nodes of row r's weighted rule (oracle.rules, boundary classes R1) at which
  the weight is nonzero (the p=2 stiffness middle node, where B'_r = 0, costs nothing: R2);
  Newton-Cotes: the knots and element midpoints of supp B_r at which the weight B_r (B'_r)
  is nonzero (a point where the weight vanishes contributes nothing to the row);
* a tensor row costs the product of its directions' counts, so a full mesh costs
  (sum_r count(r))^d.
"""
import numpy as np

from . import rules, spline


def _nonzero(t, p, N, r, x, order):
    cnt = 0
    for o in range(-p, p + 1):
        j = r + o
        if 0 <= j < N:
            v = spline.basis_scalar(t, j, p, x) if order == 0 else spline.deriv_scalar(t, j, p, x, 1)
            cnt += abs(v) > 1e-12
    return cnt


def row_counts(p, n, kind="mass", mode="gauss"):
    """Per 1D row r (unit spacing, n elements): (Gaussian count, Newton-Cotes count)."""
    order = 0 if kind == "mass" else 1
    t = spline.open_uniform_knots(p, n, length=float(n))
    N = n + p
    R = rules.rules_1d(p, n, kind, mode)
    out = []
    for r in range(N):
        xs = np.asarray(R[r].x) * n                        # unit-spacing node positions
        weight = (lambda x: spline.basis_scalar(t, r, p, x)) if order == 0 else (lambda x: spline.deriv_scalar(t, r, p, x, 1))
        g = sum(_nonzero(t, p, N, r, x, order) for x in xs if abs(weight(x)) > 1e-12)
        a, b = t[r], t[r + p + 1]
        pts = sorted(set([float(k) for k in range(int(a), int(b) + 1)] + [k + 0.5 for k in range(int(a), int(b))]))
        nc = 0
        for x in pts:
            w = spline.basis_scalar(t, r, p, x) if order == 0 else spline.deriv_scalar(t, r, p, x, 1)
            if abs(w) > 1e-12:
                nc += _nonzero(t, p, N, r, x, order)
        out.append((g, nc))
    return out


def mesh_counts(p, n, d, kind="mass", mode="gauss"):
    """Total evaluations over the n^d-element mesh: (Gaussian, Newton-Cotes)."""
    rc = row_counts(p, n, kind, mode)
    return sum(g for g, _ in rc) ** d, sum(c for _, c in rc) ** d
