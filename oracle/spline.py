"""B-spline basis on open uniform knot vectors -- ORACLE (test infrastructure only).

P:116-123 (eq:Gmap3): the knot vector has p+1 copies of each end point and simple
interior knots (maximal continuity C^{p-1}).  P:130-131 (eq:DimUni): the space has
dim = p + n_EL basis functions.  The basis is the textbook Cox-de Boor recursion,
written out literally (no table tricks), right-continuous except at the right end
point of the knot span, where it is left-continuous (reading R10).

Parity pinned by tests/test_oracle_spline.py against scipy.interpolate.BSpline,
partition of unity and the SPEC example values.
"""
import numpy as np


def open_uniform_knots(p, n, length=1.0):
    """Open uniform knot vector of eq:Gmap3 on [0, length] with n elements."""
    inner = [length * k / n for k in range(1, n)]
    return np.array([0.0] * (p + 1) + inner + [float(length)] * (p + 1), dtype=np.float64)


def dim(p, n):
    """eq:DimUni: dim S = p + n_EL."""
    return p + n


def _zeroth(t, i, x):
    """B_{i,0}: indicator of [t_i, t_{i+1}), closed at the right end of the span."""
    x = np.asarray(x, dtype=np.float64)
    lo, hi = t[i], t[i + 1]
    if hi <= lo:
        return np.zeros_like(x)
    out = ((x >= lo) & (x < hi)).astype(np.float64)
    if hi == t[-1]:                      # left-continuous at the right end point
        out = np.where(x == hi, 1.0, out)
    return out


def _frac(num, den):
    return 0.0 if den == 0.0 else num / den


def basis(t, i, k, x):
    """Cox-de Boor: B_{i,k}(x) for knot vector t (0/0 := 0)."""
    if k == 0:
        return _zeroth(t, i, x)
    x = np.asarray(x, dtype=np.float64)
    left_den = t[i + k] - t[i]
    right_den = t[i + k + 1] - t[i + 1]
    out = np.zeros_like(x)
    if left_den != 0.0:
        out = out + (x - t[i]) / left_den * basis(t, i, k - 1, x)
    if right_den != 0.0:
        out = out + (t[i + k + 1] - x) / right_den * basis(t, i + 1, k - 1, x)
    return out


def deriv(t, i, k, x, order=1):
    """order-th derivative of B_{i,k}: B' = k/(t_{i+k}-t_i) B_{i,k-1} - k/(t_{i+k+1}-t_{i+1}) B_{i+1,k-1}."""
    if order == 0:
        return basis(t, i, k, x)
    x = np.asarray(x, dtype=np.float64)
    if k == 0:
        return np.zeros_like(x)
    out = np.zeros_like(x)
    left_den = t[i + k] - t[i]
    right_den = t[i + k + 1] - t[i + 1]
    if left_den != 0.0:
        out = out + k / left_den * deriv(t, i, k - 1, x, order - 1)
    if right_den != 0.0:
        out = out - k / right_den * deriv(t, i + 1, k - 1, x, order - 1)
    return out


def support(t, i, k):
    """supp B_{i,k} = [t_i, t_{i+k+1}] (reading R11 of the garbled P:223)."""
    return float(t[i]), float(t[i + k + 1])


def interacting(p, n, j):
    """Indices i with |supp B_i cap supp B_j| > 0: {j-p..j+p} clipped to [0, dim)."""
    return [i for i in range(j - p, j + p + 1) if 0 <= i < dim(p, n)]


def basis_scalar(t, i, k, x):
    """Cox-de Boor for one scalar x of any real type (float or mpmath.mpf); same
    conventions as ``basis`` (used to refine the rules in high precision)."""
    if k == 0:
        lo, hi = t[i], t[i + 1]
        if hi <= lo:
            return 0 * x
        if lo <= x < hi or (x == hi and hi == t[-1]):
            return 0 * x + 1
        return 0 * x
    out = 0 * x
    if t[i + k] != t[i]:
        out += (x - t[i]) / (t[i + k] - t[i]) * basis_scalar(t, i, k - 1, x)
    if t[i + k + 1] != t[i + 1]:
        out += (t[i + k + 1] - x) / (t[i + k + 1] - t[i + 1]) * basis_scalar(t, i + 1, k - 1, x)
    return out


def deriv_scalar(t, i, k, x, order=1):
    """order-th derivative of B_{i,k} at a scalar x of any real type."""
    if order == 0:
        return basis_scalar(t, i, k, x)
    if k == 0:
        return 0 * x
    out = 0 * x
    if t[i + k] != t[i]:
        out += k / (t[i + k] - t[i]) * deriv_scalar(t, i, k - 1, x, order - 1)
    if t[i + k + 1] != t[i + 1]:
        out -= k / (t[i + k + 1] - t[i + 1]) * deriv_scalar(t, i + 1, k - 1, x, order - 1)
    return out
