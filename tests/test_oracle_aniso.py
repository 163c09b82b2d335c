"""Pins for the oracle on meshes with a different element count per direction (eq:Gmap3,
P:113-120: each parameter direction has its own knot vector with n_EL^i elements; eq:DimMulti,
P:134-136).  Independent references: the exact c = 1 Galerkin matrices as Kronecker products
of per-direction 1D matrices built with scipy (tests/wgq_exact.py), exact integrals of
multilinear fields against the basis, and the row-independence of the generated field."""
import numpy as np
import pytest
from scipy.integrate import quad
from scipy.interpolate import BSpline

import inputs
from oracle import assemble, operators
from wgq_exact import exact_nd, to_ell


@pytest.mark.parametrize("p,n,d", [(2, (3, 5, 4), 3), (3, (4, 6), 2), (3, (3, 4, 5), 3), (2, (2, 7), 2)])
def test_constant_coefficient_is_kronecker_galerkin(p, n, d):
    rows = np.arange(int(np.prod([na + p for na in n])))
    A = assemble.assemble_rows(p, n, d, rows, {"kind": "const", "c0": 1.0})
    M, K = exact_nd(p, n, d)
    for name, B in (("mass", M), ("stiffness", K)):
        ref = to_ell(B, p, n, d)
        assert np.max(np.abs(A[name] - ref)) < 1e-14 * np.max(np.abs(ref)), name


def _int_B(p, n):
    t = np.array([0.0] * (p + 1) + [k / n for k in range(1, n)] + [1.0] * (p + 1))
    return np.array([(t[j + p + 1] - t[j]) / (p + 1) for j in range(n + p)])


def _int_xB(p, n):
    t = np.array([0.0] * (p + 1) + [k / n for k in range(1, n)] + [1.0] * (p + 1))
    out = []
    for j in range(n + p):
        b = BSpline.basis_element(t[j:j + p + 2], extrapolate=False)
        out.append(sum(quad(lambda x: x * np.nan_to_num(b(x)), t[e], t[e + 1], epsabs=1e-16, epsrel=1e-14)[0]
                       for e in range(j, j + p + 1) if t[e + 1] > t[e]))
    return np.array(out)


@pytest.mark.parametrize("p,n", [(3, (4, 6, 5)), (2, (6, 3, 4))])
def test_load_of_multilinear_field_exact_aniso(p, n):
    """f = x y z on an anisotropic vertex grid (vertex j of direction a at j / n_a) is
    reproduced by the interpolant, and every mass rule integrates it against B_i exactly."""
    d = 3
    Ns = [na + p for na in n]
    rows = np.arange(int(np.prod(Ns)))
    z, y, x = np.meshgrid(np.arange(n[2] + 1) / n[2], np.arange(n[1] + 1) / n[1], np.arange(n[0] + 1) / n[0],
                          indexing="ij")
    b = operators.load_rows(p, n, d, rows, {"kind": "grid"}, grid=x * y * z)
    IX = [_int_xB(p, na) for na in n]
    ref = np.array([np.prod([IX[a][i] for a, i in enumerate(assemble.decode(int(r), Ns, d))]) for r in rows])
    assert np.max(np.abs(b - ref)) < 1e-14 * np.max(np.abs(ref))
    b1 = operators.load_rows(p, n, d, rows, {"kind": "const", "c0": 1.0})
    I = [_int_B(p, na) for na in n]
    ref1 = np.array([np.prod([I[a][i] for a, i in enumerate(assemble.decode(int(r), Ns, d))]) for r in rows])
    assert np.max(np.abs(b1 - ref1) / ref1) < 1e-13


def test_aniso_grid_field_slab_equals_global():
    n = (7, 5, 6)
    full = inputs.lognormal_grid(n, seed=3, dim=3)
    assert full.shape == (7, 6, 8)
    part = inputs.lognormal_grid(n, seed=3, dim=3, plane0=2, planes=3)
    assert np.array_equal(part, full[2:5])
    iso = inputs.lognormal_grid(6, seed=3, dim=3)
    assert np.array_equal(iso, inputs.lognormal_grid((6, 6, 6), seed=3, dim=3))
    two = inputs.lognormal_grid((9, 4), seed=3, dim=2)
    assert two.shape == (5, 10)


@pytest.mark.parametrize("p,n,d", [(3, (5, 7), 2), (2, (3, 4, 5), 3)])
def test_variable_coefficient_row_identities_aniso(p, n, d):
    """P9 on an anisotropic mesh for a variable coefficient: K 1 = 0 and M 1 = sum_k W^M."""
    Ns = [na + p for na in n]
    rows = np.arange(int(np.prod(Ns)))
    desc = inputs.coefficient({"kind": "fourier_logn", "seed": 4, "n_modes": 8, "amp": 0.3}, d)
    A = assemble.assemble_rows(p, n, d, rows, desc)
    m1, mx, kx = assemble.row_weight_sums(p, n, d, rows, desc)
    assert np.max(np.abs(A["stiffness"].sum(axis=1)) / np.abs(A["stiffness"]).max(axis=1)) < 1e-13
    assert np.max(np.abs(A["mass"].sum(axis=1) - m1) / m1) < 1e-13
