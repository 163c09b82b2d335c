"""Load vector and matrix-free operator application -- ORACLE (test infrastructure only).

SURVEY §8(f) rows 1 and 2, written from the paper's definitions:

* Load vector (eq:Load, J = I):  b_i = int f B_i dx.  Row i uses its own mass-kind
  weighted rule (the measure B_i, eq:GaussQuadSys P:249-252), i.e. the same node tensor and
  effective weights w^M = omega B_{i_a}(x) as row i of the mass matrix:

      b_i = sum_k [prod_a w^M_{i_a,k_a}] f(x^M_k)

  evaluated literally over the node tensor.

* Matrix-free application (the consumer of the row-wise scheme named at P:63-64):
  y = A u for A = M or K as *defined* by the row rules (oracle.assemble), computed by the
  plain definition y_i = sum_j A_ij u_j over the row's ELL columns.
"""
import numpy as np

from . import assemble, coeff


def load_rows(p, n, d, rows, desc, grid=None, plane0=0, mode="gauss"):
    """b_i for the requested global rows (f given by a coefficient descriptor)."""
    ns = assemble.dims(n, d)
    tabs = [assemble.tables_1d(p, na, mode) for na in ns]
    Ns = [na + p for na in ns]
    out = np.zeros(len(rows))
    for ri, row in enumerate(rows):
        idx = assemble.decode(int(row), Ns, d)
        R = [tabs[a][i] for a, i in enumerate(idx)]
        X = np.meshgrid(*[r.xM for r in R], indexing="ij")
        W = coeff.evaluate(desc, n, X, grid, plane0)
        for a in range(d):
            shape = [1] * d
            shape[a] = -1
            W = W * R[a].wM.reshape(shape)
        out[ri] = W.sum()
    return out


def apply_rows(p, n, d, rows, desc, u, kind, grid=None, plane0=0, mode="gauss"):
    """y_i = sum_j A_ij u_j (A = 'mass' or 'stiffness') for the requested global rows; u is
    the full coefficient vector (length N^d, global row order)."""
    A = assemble.assemble_rows(p, n, d, rows, desc, kinds=(kind,), grid=grid, plane0=plane0, mode=mode)[kind]
    y = np.zeros(len(rows))
    for ri, row in enumerate(rows):
        cols = assemble.ell_columns(p, n, d, int(row))
        ok = cols >= 0
        y[ri] = A[ri][ok] @ u[cols[ok]]
    return y
