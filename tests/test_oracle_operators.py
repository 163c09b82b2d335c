"""Pins for oracle/operators.py (no GPU): the load vector (eq:Load) and the
matrix-free product y = A u.

Load vector: the mass-kind rule of row i is exact on the spline space interacting with
B_i, which contains the constants and the linear functions (partition of unity / linear
reproduction), so for f = c0, f = x_a and the bilinear f = x y the rule returns the exact
integrals int f B_i, computed here independently (closed form int B_j, scipy quad) —
SPEC S:345-348.  A multilinear GRID field reproduces such f exactly at every point.
Application: for c == 1 the rule-defined matrices are the exact Galerkin matrices,
so y = A u must equal the Kronecker-product matrices of tests/wgq_exact.py times u; for
variable c the P9 identities (K 1 = 0, M g^a = sum_k W^M x^a) pin it on every row.
"""
import numpy as np
import pytest
from scipy.integrate import quad
from scipy.interpolate import BSpline

import inputs
from oracle import assemble, operators
from wgq_exact import exact_nd


def knots(p, n):
    return np.array([0.0] * (p + 1) + [k / n for k in range(1, n)] + [1.0] * (p + 1))


def int_B(p, n):
    """int_0^1 B_j = (t_{j+p+1} - t_j) / (p+1) for all j (the textbook identity)."""
    t = knots(p, n)
    return np.array([(t[j + p + 1] - t[j]) / (p + 1) for j in range(n + p)])


def int_xB(p, n):
    """int_0^1 x B_j(x) dx by adaptive quadrature on each knot span."""
    t = knots(p, n)
    out = []
    for j in range(n + p):
        b = BSpline.basis_element(t[j:j + p + 2], extrapolate=False)
        tot = 0.0
        for e in range(j, j + p + 1):
            if t[e + 1] > t[e]:
                tot += quad(lambda x: x * np.nan_to_num(b(x)), t[e], t[e + 1], epsabs=1e-16, epsrel=1e-14)[0]
        out.append(tot)
    return np.array(out)


def vertex_field(n, d, f):
    """Vertex values [z][y][x] (x fastest) of f at the vertices (a, b, c) / n."""
    ax = np.arange(n + 1) / n
    if d == 1:
        return f(ax)
    if d == 2:
        Y, X = np.meshgrid(ax, ax, indexing="ij")
        return f(X, Y)
    Z, Y, X = np.meshgrid(ax, ax, ax, indexing="ij")
    return f(X, Y, Z)


CASES = [(2, 1, 7), (3, 1, 9), (2, 2, 5), (3, 2, 4), (2, 3, 3), (3, 3, 3)]


@pytest.mark.parametrize("p,d,n", CASES)
def test_load_constant_is_integral_of_basis(p, d, n):
    N = n + p
    rows = np.arange(N ** d)
    b = operators.load_rows(p, n, d, rows, {"kind": "const", "c0": 1.75})
    I = int_B(p, n)
    ref = np.array([1.75 * np.prod([I[i] for i in assemble.decode(int(r), N, d)]) for r in rows])
    assert np.max(np.abs(b - ref) / np.abs(ref)) < 1e-13


@pytest.mark.parametrize("p,d,n", CASES)
def test_load_linear_fields_are_exact(p, d, n):
    N = n + p
    rows = np.arange(N ** d)
    I, IX = int_B(p, n), int_xB(p, n)
    fields = [(lambda *x: x[0], [IX] + [I] * (d - 1))]
    if d >= 2:
        fields.append((lambda *x: x[1], [I, IX] + [I] * (d - 2)))
        fields.append((lambda *x: x[0] * x[1], [IX, IX] + [I] * (d - 2)))
    if d == 3:
        fields.append((lambda *x: x[2], [I, I, IX]))
        fields.append((lambda *x: x[0] * x[2], [IX, I, IX]))
        fields.append((lambda *x: x[1] * x[2], [I, IX, IX]))
        fields.append((lambda *x: x[0] * x[1] * x[2], [IX, IX, IX]))
    for f, factors in fields:
        grid = vertex_field(n, d, f)
        b = operators.load_rows(p, n, d, rows, {"kind": "grid"}, grid=grid)
        ref = np.array([np.prod([factors[a][i] for a, i in enumerate(assemble.decode(int(r), N, d))]) for r in rows])
        assert np.max(np.abs(b - ref)) < 1e-14 * np.max(np.abs(ref))


@pytest.mark.parametrize("p,d,n", [(2, 2, 5), (3, 3, 3)])
def test_load_equals_mass_row_sums(p, d, n):
    """b(f) = M(c = f) 1 by partition of unity (a cross-check of two oracle code paths)."""
    N = n + p
    rows = np.arange(N ** d)
    desc = inputs.coefficient({"kind": "fourier_logn", "seed": 3, "n_modes": 8, "amp": 0.3}, d)
    b = operators.load_rows(p, n, d, rows, desc)
    M = assemble.assemble_rows(p, n, d, rows, desc, kinds=("mass",))["mass"]
    assert np.max(np.abs(b - M.sum(axis=1)) / np.abs(b)) < 1e-13


@pytest.mark.parametrize("p,d,n", [(2, 1, 8), (3, 2, 4), (2, 3, 3), (3, 3, 3)])
def test_apply_constant_coefficient_is_galerkin_product(p, d, n):
    N = n + p
    rows = np.arange(N ** d)
    u = np.random.default_rng(1).standard_normal(N ** d)
    M, K = exact_nd(p, n, d)
    for kind, A in (("mass", M), ("stiffness", K)):
        y = operators.apply_rows(p, n, d, rows, {"kind": "const", "c0": 1.0}, u, kind)
        ref = A @ u
        assert np.linalg.norm(y - ref) < 1e-13 * np.linalg.norm(ref), kind


@pytest.mark.parametrize("p,d,n", [(2, 2, 5), (3, 3, 3)])
def test_apply_full_coverage_identities(p, d, n):
    """P9 on y = A u: K 1 = 0 and M g^a = sum_k W^M x^a, for a variable coefficient."""
    N = n + p
    rows = np.arange(N ** d)
    desc = inputs.coefficient({"kind": "fourier_logn", "seed": 5, "n_modes": 8, "amp": 0.3}, d)
    one = np.ones(N ** d)
    yk = operators.apply_rows(p, n, d, rows, desc, one, "stiffness")
    ym = operators.apply_rows(p, n, d, rows, desc, one, "mass")
    assert np.max(np.abs(yk)) < 1e-13 * np.max(np.abs(ym)) * n * n
    m1, mx, _ = assemble.row_weight_sums(p, n, d, rows, desc)
    assert np.max(np.abs(ym - m1) / m1) < 1e-13
    g = assemble.greville(p, n)
    for a in range(d):
        ga = np.array([g[assemble.decode(int(r), N, d)[a]] for r in range(N ** d)])
        y = operators.apply_rows(p, n, d, rows, desc, ga, "mass")
        assert np.max(np.abs(y - mx[:, a]) / np.abs(m1)) < 1e-13


@pytest.mark.parametrize("p,n,z0,z1", [(2, 6, 3, 5), (3, 6, 4, 8), (3, 7, 0, 2), (2, 5, 5, 6)])
def test_load_multilinear_fields_on_a_slab(p, n, z0, z1):
    """The same exact integrals from a slab of vertex planes (plane0 != 0): rows of z-planes
    [z0, z1] need vertex planes [max(0, z0 - p), min(n, z1 + 1)] only."""
    d, N = 3, n + p
    rows = np.arange(z0 * N * N, (z1 + 1) * N * N)
    lo, hi = max(0, z0 - p), min(n, z1 + 1)
    I, IX = int_B(p, n), int_xB(p, n)
    for f, fac in ((lambda x, y, z: z, (I, I, IX)), (lambda x, y, z: x * y * z, (IX, IX, IX)),
                   (lambda x, y, z: 1.0 + y * z, None)):
        grid = vertex_field(n, d, f)[lo:hi + 1]
        b = operators.load_rows(p, n, d, rows, {"kind": "grid"}, grid=grid, plane0=lo)
        if fac is None:
            ref = np.array([I[i] * I[j] * I[k] + I[i] * IX[j] * IX[k]
                            for i, j, k in (assemble.decode(int(r), N, d) for r in rows)])
        else:
            ref = np.array([np.prod([fac[a][i] for a, i in enumerate(assemble.decode(int(r), N, d))]) for r in rows])
        assert np.max(np.abs(b - ref)) < 1e-14 * np.max(np.abs(ref))
