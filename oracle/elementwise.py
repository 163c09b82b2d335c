"""Standard element-wise Gauss-Legendre assembly -- ORACLE (test infrastructure only).

The paper's comparison scheme: loop over elements, (p+1)^d Gauss-
Legendre points per element, scatter B_i B_j (mass) and grad B_i . grad B_j
(stiffness, J = I) into a dense matrix.  Exact for c == 1 (degree 2p per direction).
Only used on tiny meshes as an independent check of the row-wise rules.
"""
import numpy as np

from . import coeff, quadrature, spline


def assemble_dense(p, n, d, desc, kinds=("mass", "stiffness"), m=None, grid=None, plane0=0):
    if m is None:
        m = p + 1
    t = spline.open_uniform_knots(p, n)
    N = n + p
    h = 1.0 / n
    nd = N ** d
    out = {k: np.zeros((nd, nd)) for k in kinds}
    gx, gw = quadrature.gauss_legendre(m, 0.0, 1.0)
    for e in np.ndindex(*([n] * d)):
        # per direction: points, weights, values / derivatives of the p+1 functions e..e+p
        pts, wts, V, D = [], [], [], []
        for a in range(d):
            x = h * (e[a] + gx)
            pts.append(x)
            wts.append(h * gw)
            V.append(np.array([spline.basis(t, e[a] + l, p, x) for l in range(p + 1)]))
            D.append(np.array([spline.deriv(t, e[a] + l, p, x, 1) for l in range(p + 1)]))
        X = np.meshgrid(*pts, indexing="ij")
        c = coeff.evaluate(desc, n, X, grid, plane0)
        Wq = c.copy()
        for a in range(d):
            shape = [1] * d
            shape[a] = m
            Wq = Wq * wts[a].reshape(shape)
        gidx = np.zeros([p + 1] * d, dtype=np.int64)
        for li in np.ndindex(*([p + 1] * d)):
            gidx[li] = sum((e[a] + li[a]) * N ** a for a in range(d))
        gidx = gidx.reshape(-1)
        # local element matrices: sum over the (p+1)^d GL points of the integrand
        q = "xyz"[:d]
        li = "abc"[:d]
        lj = "def"[:d]
        ops_m = [Wq] + [V[a] for a in range(d)] + [V[a] for a in range(d)]
        spec_m = q + "," + ",".join(li[a] + q[a] for a in range(d)) + "," + ",".join(lj[a] + q[a] for a in range(d)) + "->" + li + lj
        nl = (p + 1) ** d
        if "mass" in out:
            loc = np.einsum(spec_m, *ops_m).reshape(nl, nl)
            out["mass"][np.ix_(gidx, gidx)] += loc
        if "stiffness" in out:
            loc = np.zeros((nl, nl))
            for a in range(d):
                T = [D[b] if b == a else V[b] for b in range(d)]
                loc += np.einsum(spec_m, *([Wq] + T + T)).reshape(nl, nl)
            out["stiffness"][np.ix_(gidx, gidx)] += loc
    return out


def dense_to_ell(A, p, n, d):
    """ELL rows (slot order of assemble.py) of a dense N^d x N^d matrix."""
    from .assemble import ell_columns
    nd = A.shape[0]
    s = 2 * p + 1
    out = np.zeros((nd, s ** d))
    for r in range(nd):
        cols = ell_columns(p, n, d, r)
        ok = cols >= 0
        out[r, ok] = A[r, cols[ok]]
    return out
