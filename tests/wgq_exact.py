"""Exact c = 1 Galerkin matrices built independently with scipy (test helper, no GPU)."""
import numpy as np
from scipy.interpolate import BSpline
from scipy.special import roots_legendre


def exact_1d(p, n):
    """Exact 1D mass/stiffness (c = 1) with scipy: per-element (p+2)-point GL."""
    t = np.array([0.0] * (p + 1) + [k / n for k in range(1, n)] + [1.0] * (p + 1))
    N = n + p
    funcs = []
    for i in range(N):
        c = np.zeros(N)
        c[i] = 1.0
        funcs.append(BSpline(t, c, p, extrapolate=False))
    xg, wg = roots_legendre(p + 2)
    M = np.zeros((N, N))
    K = np.zeros((N, N))
    for e in range(n):
        a, b = e / n, (e + 1) / n
        x = 0.5 * (b - a) * xg + 0.5 * (a + b)
        w = 0.5 * (b - a) * wg
        ids = list(range(e, e + p + 1))          # the p+1 functions nonzero on element e
        V = np.array([np.nan_to_num(funcs[i](x)) for i in ids])
        D = np.array([np.nan_to_num(funcs[i].derivative(1)(x)) for i in ids])
        M[np.ix_(ids, ids)] += (V * w) @ V.T
        K[np.ix_(ids, ids)] += (D * w) @ D.T
    return M, K


def exact_nd(p, n, d):
    M1, K1 = exact_1d(p, n)
    M = M1
    for _ in range(d - 1):
        M = np.kron(M1, M)
    K = np.zeros_like(M)
    for a in range(d):
        T = None
        for b in range(d):          # row index i = i1 + N i2 + N^2 i3 -> kron(dir d-1, ..., dir 0)
            f = K1 if b == a else M1
            T = f if T is None else np.kron(f, T)
        K += T
    return M, K


def to_ell(A, p, n, d):
    N = n + p
    s = 2 * p + 1
    out = np.zeros((N ** d, s ** d))
    for r in range(N ** d):
        ir = [(r // N ** a) % N for a in range(d)]
        for slot in range(s ** d):
            o = [(slot // s ** a) % s - p for a in range(d)]
            j = [ir[a] + o[a] for a in range(d)]
            if all(0 <= j[a] < N for a in range(d)):
                out[r, slot] = A[r, sum(j[a] * N ** a for a in range(d))]
    return out
