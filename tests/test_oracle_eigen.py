"""Pins for oracle/eigen.py (no GPU): experiments E1/E2 of sec:NUMER.

* the exact spectrum is the textbook π² Σ k_a² (multiplicities: the 10th eigenvalue is 17π² in
  2D and 11π² in 3D);
* for c == 1 the oracle's weighted-rule spectrum equals the spectrum of the exact Galerkin
  matrices built independently with scipy (wgq_exact), and of the oracle's element-wise GL
  scheme ("almost identical error when compared to the standard Gauss integration");
* the discrete eigenvalues converge to the exact ones at the Galerkin rate 2p (P:470-471:
  "close to the theoretical order of 2p") and from above (Rayleigh-Ritz: min-max).
"""
import numpy as np
import pytest

from oracle import eigen, elementwise
from wgq_exact import exact_nd


def test_exact_spectrum_multiplicities():
    pi2 = np.pi ** 2
    assert np.allclose(eigen.exact_eigenvalues(1, 12), pi2 * np.arange(1, 13) ** 2)
    e2 = eigen.exact_eigenvalues(2, 10) / pi2
    assert np.allclose(e2, [2, 5, 5, 8, 10, 10, 13, 13, 17, 17])
    e3 = eigen.exact_eigenvalues(3, 10) / pi2
    assert np.allclose(e3, [3, 6, 6, 6, 9, 9, 9, 11, 11, 11])


@pytest.mark.parametrize("p,d,n", [(2, 1, 12), (3, 1, 12), (2, 2, 5), (3, 2, 5)])
def test_weighted_spectrum_equals_exact_galerkin(p, d, n):
    lam = eigen.spectrum(p, n, d)
    M, K = exact_nd(p, n, d)
    ref = eigen.discrete_eigenvalues(K, M, p, n, d)
    assert lam.shape == ref.shape == ((n + p - 2) ** d,)
    assert np.max(np.abs(lam - ref) / ref) < 1e-12
    G = elementwise.assemble_dense(p, n, d, {"kind": "const", "c0": 1.0})
    gl = eigen.discrete_eigenvalues(G["stiffness"], G["mass"], p, n, d)
    assert np.max(np.abs(lam - gl) / gl) < 1e-12


@pytest.mark.parametrize("p", [2, 3])
def test_1d_convergence_rate_2p(p):
    ex = eigen.exact_eigenvalues(1, 3)
    errs = []
    for n in (8, 16, 32):
        lam = eigen.spectrum(p, n, 1)[:3]
        assert np.all(lam >= ex * (1 - 1e-13))          # Rayleigh-Ritz upper bounds
        errs.append(lam[1] / ex[1] - 1)
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(rates - 2 * p) < 0.3), rates


@pytest.mark.parametrize("p", [2, 3])
def test_2d_tenth_eigenvalue_rate(p):
    """fig:Result2DConvergence (left): the 10th eigenvalue of the 2D problem."""
    ex = eigen.exact_eigenvalues(2, 10)[9]
    errs = [eigen.spectrum(p, n, 2)[9] / ex - 1 for n in (8, 16, 24)]
    assert min(errs) > 0
    rates = [np.log(errs[0] / errs[1]) / np.log(2), np.log(errs[1] / errs[2]) / np.log(1.5)]
    assert abs(rates[-1] - 2 * p) < 0.8, rates
