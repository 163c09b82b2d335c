"""Generalised eigenvalue validation (experiments E1/E2) -- ORACLE (test infrastructure only).

SURVEY §8(f) row 4; PAPER.md sec:NUMER.  The paper validates the rules on the
elliptic eigenvalue problem  -Δu = λu  on [0,1]^d discretised with the assembled matrices:

* E1 (fig:ResultComparison): 1D, 1000 uniform elements, p = 2, 3; the discrete
  spectra from the weighted rules and from standard Gauss integration are "almost
  identical", the matrix entries differing by ~1e-15.
* E2 (fig:Result2DConvergence): the 10th eigenvalue of the 2D and 3D problems
  converges at a rate "close to the theoretical order of 2p".

Readings (R15): homogeneous Dirichlet conditions, imposed by dropping the basis
functions that do not vanish on the boundary (index 0 or N-1 in some direction; open knot
vectors make the basis interpolatory at the ends), so the discrete problem is
K_II v = λ M_II v on the remaining indices I.  The exact eigenvalues are the textbook
λ = π² Σ_a k_a², k_a ≥ 1, counted with multiplicity (the 10th is 17π² in 2D, 11π² in 3D).

Every step is a plain definition: dense matrices from the ELL rows of ``assemble`` and
scipy's generalised symmetric eigensolver (a library primitive).
"""
import itertools

import numpy as np
import scipy.linalg

from . import assemble


def ell_to_dense(E, p, n, d):
    """Dense N^d x N^d matrix from ELL rows in assemble.py's slot order."""
    N = n + p
    A = np.zeros((N ** d, N ** d))
    for r in range(N ** d):
        cols = assemble.ell_columns(p, n, d, r)
        ok = cols >= 0
        A[r, cols[ok]] = E[r, ok]
    return A


def interior_indices(p, n, d):
    """Rows i = i_1 + N i_2 + ... whose every index lies in [1, N-2] (Dirichlet)."""
    N = n + p
    keep = []
    for r in range(N ** d):
        idx = assemble.decode(r, N, d)
        if all(1 <= i <= N - 2 for i in idx):
            keep.append(r)
    return np.array(keep, dtype=np.int64)


def exact_eigenvalues(d, count):
    """The `count` smallest Dirichlet Laplacian eigenvalues on [0,1]^d, with multiplicity."""
    kmax = count          # (k, 1, ..., 1), k = 1..count, are count values below any k_a > count
    vals = sorted(np.pi ** 2 * sum(k * k for k in ks) for ks in itertools.product(range(1, kmax + 1), repeat=d))
    return np.array(vals[:count])


def discrete_eigenvalues(K, M, p, n, d):
    """Ascending eigenvalues of K_II v = λ M_II v (symmetric K, M)."""
    I = interior_indices(p, n, d)
    return scipy.linalg.eigh(K[np.ix_(I, I)], M[np.ix_(I, I)], eigvals_only=True)


def spectrum(p, n, d, desc=None, mode="gauss"):
    """Discrete Dirichlet spectrum of the row-wise weighted assembly (c from `desc`, default 1)."""
    desc = desc or {"kind": "const", "c0": 1.0}
    N = n + p
    A = assemble.assemble_rows(p, n, d, np.arange(N ** d), desc, mode=mode)
    return discrete_eigenvalues(ell_to_dense(A["stiffness"], p, n, d), ell_to_dense(A["mass"], p, n, d), p, n, d)
