"""Eigenvalue validation of the assembled matrices (experiments E1/E2).

PAPER.md sec:NUMER: -Δu = λu on [0,1]^d with homogeneous Dirichlet conditions,
K_II v = λ M_II v on the basis functions that vanish on the boundary (R15).  The
matrices come from libwgq's CSR assembly (the CUDA kernels); the dense generalised
eigensolve is a library call (torch.linalg: Cholesky of M_II, the congruent standard
problem L⁻¹ K_II L⁻ᵀ, eigvalsh) on the same device.  This is a validation tool for the
small meshes of the paper's experiments (dense N^d x N^d), not part of the assembly path.
"""
import itertools
import math
import warnings

import torch

from . import api


def dirichlet_index(rules, device="cuda"):
    """Global rows whose every index lies in [1, N-2] (ascending)."""
    N, d = rules.N, rules.dim
    r = torch.arange(N ** d, device=device)
    keep = torch.ones_like(r, dtype=torch.bool)
    for a in range(d):
        i = (r // N ** a) % N
        keep &= (i >= 1) & (i <= N - 2)
    return r[keep]


def dense_matrices(rules, coeff, stream=None):
    """(M, K) as dense FP64 device matrices, assembled by libwgq in CSR layout."""
    row_ptr, col_idx, vals = api.assemble_csr(rules, coeff, ("mass", "stiffness"), stream=stream)
    n = rules.n_rows
    out = []
    for k in ("mass", "stiffness"):
        with warnings.catch_warnings():
            warnings.filterwarnings("ignore", message="Sparse CSR tensor support is in beta")
            A = torch.sparse_csr_tensor(row_ptr, col_idx.long(), vals[k], (n, n), dtype=torch.float64,
                                        check_invariants=True)       # also validates the CSR structure
        out.append(A.to_dense())
    return tuple(out)


def generalized_eigenvalues(K, M):
    """Ascending eigenvalues of K v = λ M v for symmetric K and symmetric positive definite M."""
    L = torch.linalg.cholesky(M)
    X = torch.linalg.solve_triangular(L, K, upper=False)
    C = torch.linalg.solve_triangular(L, X.mT, upper=False)
    return torch.linalg.eigvalsh(0.5 * (C + C.mT))


def spectrum(rules, coeff):
    """Discrete Dirichlet spectrum (ascending) of the weighted-rule assembly on rules' mesh.
    Symmetric matrices are required (constant coefficient, R4)."""
    M, K = dense_matrices(rules, coeff)
    I = dirichlet_index(rules, M.device)
    return generalized_eigenvalues(K[I][:, I], M[I][:, I])


def exact_eigenvalues(d, count):
    """The `count` smallest eigenvalues π² Σ k_a² (k_a ≥ 1) of the Dirichlet Laplacian on [0,1]^d."""
    kmax = count          # (k, 1, ..., 1), k = 1..count, are count values below any k_a > count
    vals = sorted(math.pi ** 2 * sum(k * k for k in ks) for ks in itertools.product(range(1, kmax + 1), repeat=d))
    return vals[:count]
