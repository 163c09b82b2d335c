"""Pins for oracle/assemble.py (no GPU).

c == 1: the row-wise weighted assembly must equal the exact Galerkin matrices
(P:449), built here independently as Kronecker products of 1D matrices integrated
with scipy's BSpline and Gauss-Legendre (P5/P11), and the oracle's element-wise GL
scheme; P:452's 1D 1000-element comparison.  Variable c: the full-coverage identities
of SURVEY §8(c) P9, which hold for every row and any c, plus symmetry for constant c.
"""
import numpy as np
import pytest
import inputs
from oracle import assemble, elementwise
from wgq_exact import exact_1d, exact_nd, to_ell


CASES = [(2, 1, 2), (2, 1, 9), (3, 1, 3), (3, 1, 10), (2, 2, 2), (2, 2, 7), (3, 2, 3), (3, 2, 8),
         (2, 3, 2), (2, 3, 5), (3, 3, 3), (3, 3, 5)]


@pytest.mark.parametrize("p,d,n", CASES)
def test_const_coefficient_equals_exact_galerkin(p, d, n):
    N = n + p
    rows = np.arange(N ** d)
    A = assemble.assemble_rows(p, n, d, rows, {"kind": "const", "c0": 1.0})
    M, K = exact_nd(p, n, d)
    for kind, ref in (("mass", M), ("stiffness", K)):
        ref_e = to_ell(ref, p, n, d)
        rel_f = np.linalg.norm(A[kind] - ref_e) / np.linalg.norm(ref_e)
        assert rel_f < 1e-14, (kind, rel_f)
    # matches the oracle's own element-wise GL scheme as well
    if (N ** d) <= 700:
        E = elementwise.assemble_dense(p, n, d, {"kind": "const", "c0": 1.0})
        for kind in ("mass", "stiffness"):
            assert np.max(np.abs(elementwise.dense_to_ell(E[kind], p, n, d) - A[kind])) < 1e-13 * np.max(np.abs(A[kind]))


@pytest.mark.parametrize("p", [2, 3])
def test_paper_1d_1000_elements(p):
    """1D, 1000 uniform elements; weighted vs Gauss entries agree to ~1e-15
    (relative); interior rows are h * the printed mass moments."""
    n = 1000
    N = n + p
    rows = np.arange(N)
    A = assemble.assemble_rows(p, n, 1, rows, {"kind": "const", "c0": 1.0})
    M, K = exact_1d(p, n)
    for kind, ref in (("mass", M), ("stiffness", K)):
        ref_e = to_ell(ref, p, n, 1)
        assert np.max(np.abs(A[kind] - ref_e)) / np.max(np.abs(ref_e)) < 5e-13
        if kind == "mass":          # the paper's "maximum absolute difference ... of order 1e-15"
            assert np.max(np.abs(A[kind] - ref_e)) < 1e-15
    printed = {2: [1 / 120, 13 / 60, 11 / 20], 3: [1 / 5040, 1 / 42, 397 / 1680, 151 / 315]}[p]
    row = A["mass"][N // 2]
    assert np.allclose(row[:p + 1] * n, printed, rtol=1e-12, atol=0)
    assert np.allclose(row[p:] * n, printed[::-1], rtol=1e-12, atol=0)


def _coeffs(d, n):
    out = [{"kind": "const", "c0": 2.5},
           {"kind": "trig_sep", "c0": 1.0, "amp": 0.5, "trig": ("sin", "cos", "sin")[:d], "wavenum": (1, 2, 1)[:d]},
           inputs.coefficient({"kind": "fourier_logn", "seed": 7, "n_modes": 8, "amp": 0.3}, d)]
    if d >= 2:
        out.append({"kind": "grid", "grid": inputs.lognormal_grid(n, seed=11, dim=d)})
    return out


@pytest.mark.parametrize("p,d,n", [(2, 2, 6), (3, 2, 7), (2, 3, 4), (3, 3, 4)])
def test_full_coverage_identities_any_coefficient(p, d, n):
    """P9: for every row and any c, (M 1)_i = sum_k W^M_ik, (M g^a)_i = sum_k W^M_ik x^a_k,
    (K 1)_i = 0 and (K g^a)_i = sum_k W^{K,a}_ik (partition of unity + linear reproduction)."""
    N = n + p
    rows = np.arange(N ** d)
    g1 = assemble.greville(p, n)
    for desc in _coeffs(d, n):
        grid = desc.get("grid")
        A = assemble.assemble_rows(p, n, d, rows, desc, grid=grid)
        m1, mx, kx = assemble.row_weight_sums(p, n, d, rows, desc, grid=grid)
        cols = np.array([assemble.ell_columns(p, n, d, r) for r in rows])
        ok = cols >= 0
        ones = np.ones(N ** d)
        for kind in ("mass", "stiffness"):
            V = np.where(ok, A[kind], 0.0)
            scale = np.max(np.abs(V), axis=1)

            def apply(vec):
                return np.sum(V * np.where(ok, vec[np.where(ok, cols, 0)], 0.0), axis=1)

            lhs1 = apply(ones)
            rhs1 = m1 if kind == "mass" else np.zeros_like(m1)
            assert np.max(np.abs(lhs1 - rhs1) / scale) < 1e-13, (desc["kind"], kind)
            for a in range(d):
                ga = np.array([g1[(r // N ** a) % N] for r in range(N ** d)])
                rhs = mx[:, a] if kind == "mass" else kx[:, a]
                assert np.max(np.abs(apply(ga) - rhs) / scale) < 1e-13, (desc["kind"], kind, a)


@pytest.mark.parametrize("p,d,n", [(2, 2, 5), (3, 3, 3)])
def test_symmetry_only_for_constant_coefficient(p, d, n):
    """Reading R4: symmetric to rounding for constant c; O(h) asymmetric otherwise."""
    N = n + p
    rows = np.arange(N ** d)
    for desc, sym in (({"kind": "const", "c0": 3.0}, True),
                      ({"kind": "trig_sep", "c0": 1.0, "amp": 0.5, "trig": ("sin",) * d, "wavenum": (1,) * d}, False)):
        A = assemble.assemble_rows(p, n, d, rows, desc)
        for kind in ("mass", "stiffness"):
            D = np.zeros((N ** d, N ** d))
            cols = np.array([assemble.ell_columns(p, n, d, r) for r in rows])
            for r in rows:
                ok = cols[r] >= 0
                D[r, cols[r][ok]] = A[kind][r][ok]
            asym = np.max(np.abs(D - D.T)) / np.max(np.abs(D))
            assert (asym < 1e-14) if sym else (asym > 1e-6), (kind, asym)


def test_row_sums_constant_coefficient():
    """P6: c = 1 row sums: M -> prod_a int B_{i_a}, K -> 0, all rows incl. boundary."""
    p, d, n = 3, 2, 6
    N = n + p
    rows = np.arange(N ** d)
    A = assemble.assemble_rows(p, n, d, rows, {"kind": "const", "c0": 1.0})
    M1, _ = exact_1d(p, n)
    intB = M1.sum(axis=1)
    expect = np.array([intB[r % N] * intB[r // N] for r in rows])
    assert np.allclose(A["mass"].sum(axis=1), expect, rtol=1e-13, atol=0)
    assert np.max(np.abs(A["stiffness"].sum(axis=1))) < 1e-12 * n
