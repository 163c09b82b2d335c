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
    """Kronecker products of the exact 1D matrices; n an int or one count per direction."""
    ns = [n] * d if np.ndim(n) == 0 else list(n)[:d]
    one = [exact_1d(p, na) for na in ns]
    M = None
    for a in range(d):              # row index i = i1 + N1 i2 + N1 N2 i3 -> kron(dir d-1, ..., dir 0)
        M = one[a][0] if M is None else np.kron(one[a][0], M)
    K = np.zeros_like(M)
    for a in range(d):
        T = None
        for b in range(d):
            f = one[b][1] if b == a else one[b][0]
            T = f if T is None else np.kron(f, T)
        K += T
    return M, K


def to_ell(A, p, n, d):
    ns = [n] * d if np.ndim(n) == 0 else list(n)[:d]
    Ns = [na + p for na in ns]
    st = [int(np.prod(Ns[:a])) for a in range(d)]
    rows = int(np.prod(Ns))
    s = 2 * p + 1
    out = np.zeros((rows, s ** d))
    for r in range(rows):
        ir = [(r // st[a]) % Ns[a] for a in range(d)]
        for slot in range(s ** d):
            o = [(slot // s ** a) % s - p for a in range(d)]
            j = [ir[a] + o[a] for a in range(d)]
            if all(0 <= j[a] < Ns[a] for a in range(d)):
                out[r, slot] = A[r, sum(j[a] * st[a] for a in range(d))]
    return out
