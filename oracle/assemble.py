"""Row-wise weighted-Gaussian assembly, plain definition -- ORACLE (test infrastructure only).

Identity geometry on [0,1]^d (J = I: eq:Stiffness P:159-163, eq:Mass P:170-173), a
coefficient c (reading R4), tensor-product basis B_i = prod_a B_{i_a} (eq:Gmap2).  Row i
is integrated with the tensor product of its per-direction weighted rules (the
"local quadrature mask" on supp B_i; eq:Decompo P:194-199):

  M_ij = sum_k [prod_a w^M_{i_a,k_a}] c(x^M_k) prod_a B_{j_a}(x^M_{i_a,k_a})
  K_ij = sum_a sum_k [w^K_{i_a,k_a} prod_{b!=a} w^M_{i_b,k_b}] c(x^(a)_k)
                   B'_{j_a}(x^K_{i_a,k_a}) prod_{b!=a} B_{j_b}(x^M_{i_b,k_b})

with w^M = omega B_{i_a}(x), w^K = omega B'_{i_a}(x) the effective weights
and x^(a) the node tensor with stiffness nodes in direction a, mass nodes elsewhere.

Output: ELL rows of s^d = (2p+1)^d slots, slot = (o1+p) + s*((o2+p) + s*(o3+p)) with
o_a = j_a - i_a; columns outside [0, N) hold +0.0.  Rows are lexicographic with x
fastest: i = i1 + N1*(i2 + N2*i3).  Each row is evaluated literally: the full product
table prod_a B_{j_a}(x_{k_a}) (no sum factorisation) times the weight vector.

Element counts may differ per direction (n = (n_1, ..., n_d): eq:Gmap3 P:113-120 defines the
knot vector of each parameter direction by its own element count n_EL^i, and eq:DimMulti
P:134-136 the dimension N = prod_i (n_EL^i + p)); an int n means the same count in every
direction.  Each direction then has its own spacing h_a = 1/n_a, rules and tables.
"""
import numpy as np

from . import coeff, rules, spline

_TAB = {}


class Row1D:
    """Per-direction data of one 1D row r: mass and stiffness rules and the values
    of the 2p+1 neighbouring basis functions (or derivatives) at their nodes."""

    def __init__(self, xM, wM, VM, xK, wK, DK):
        self.xM, self.wM, self.VM, self.xK, self.wK, self.DK = xM, wM, VM, xK, wK, DK


def tables_1d(p, n, mode="gauss"):
    key = (p, n, mode)
    if key in _TAB:
        return _TAB[key]
    t = spline.open_uniform_knots(p, n)
    N = n + p
    RM = rules.rules_1d(p, n, "mass", mode)
    RK = rules.rules_1d(p, n, "stiffness", mode)
    out = []
    for r in range(N):
        VM = np.zeros((len(RM[r].x), 2 * p + 1))
        DK = np.zeros((len(RK[r].x), 2 * p + 1))
        for o in range(-p, p + 1):
            j = r + o
            if 0 <= j < N:
                VM[:, o + p] = spline.basis(t, j, p, RM[r].x)
                DK[:, o + p] = spline.deriv(t, j, p, RK[r].x, 1)
        out.append(Row1D(RM[r].x, RM[r].w, VM, RK[r].x, RK[r].w, DK))
    _TAB[key] = out
    return out


def dims(n, d):
    """Per-direction element counts [n_1, ..., n_d] from an int or a sequence."""
    if np.ndim(n) == 0:
        return [int(n)] * d
    ns = [int(v) for v in n]
    assert len(ns) >= d, (n, d)
    return ns[:d]


def decode(row, N, d):
    """Row index -> per-direction indices (x fastest); N an int or per-direction sizes."""
    Ns = dims(N, d)
    idx = []
    for a in range(d):
        idx.append(row % Ns[a])
        row //= Ns[a]
    return idx


def _term(dirs, desc, n, grid, plane0, absolute=False):
    """One tensor term: sum_k [prod w] c(x_k) prod_a T_a[k_a, o_a] as an ELL row
    (absolute=True: the same sum over |terms|, the rounding scale of each entry)."""
    d = len(dirs)
    xs = [x for x, _, _ in dirs]
    ws = [np.abs(w) if absolute else w for _, w, _ in dirs]
    Ts = [np.abs(T) if absolute else T for _, _, T in dirs]
    X = np.meshgrid(*xs, indexing="ij")
    c = coeff.evaluate(desc, n, X, grid, plane0)
    if absolute:
        c = np.abs(c)
    Wt = c.copy()
    for a in range(d):
        shape = [1] * d
        shape[a] = len(ws[a])
        Wt = Wt * ws[a].reshape(shape)
    # Phi[k_1..k_d, o_d, ..., o_1] = prod_a T_a[k_a, o_a]  (outer product, no summation)
    if d == 1:
        Phi = Ts[0]
    elif d == 2:
        Phi = np.einsum("ia,jb->ijba", Ts[0], Ts[1])
    else:
        Phi = np.einsum("ia,jb,kc->ijkcba", Ts[0], Ts[1], Ts[2])
    nk = Wt.size
    return Wt.reshape(nk) @ Phi.reshape(nk, -1)


def assemble_rows(p, n, d, rows, desc, kinds=("mass", "stiffness"), grid=None, plane0=0, mode="gauss",
                  absolute=False):
    """ELL values of the requested global rows: {'mass': [R, s^d], 'stiffness': [R, s^d]}.
    absolute=True returns sum_k |term_k| per entry instead (the scale of FP64 rounding in
    that entry, used by the parity tests' conditioning-aware tolerance, R12)."""
    ns = dims(n, d)
    tabs = [tables_1d(p, na, mode) for na in ns]
    Ns = [na + p for na in ns]
    s = 2 * p + 1
    out = {k: np.zeros((len(rows), s ** d)) for k in kinds}
    for ri, row in enumerate(rows):
        idx = decode(int(row), Ns, d)
        R = [tabs[a][i] for a, i in enumerate(idx)]
        if "mass" in kinds:
            out["mass"][ri] = _term([(r.xM, r.wM, r.VM) for r in R], desc, n, grid, plane0, absolute)
        if "stiffness" in kinds:
            acc = np.zeros(s ** d)
            for a in range(d):
                dirs = [(R[b].xK, R[b].wK, R[b].DK) if b == a else (R[b].xM, R[b].wM, R[b].VM) for b in range(d)]
                acc = acc + _term(dirs, desc, n, grid, plane0, absolute)
            out["stiffness"][ri] = acc
    return out


def row_weight_sums(p, n, d, rows, desc, grid=None, plane0=0, mode="gauss"):
    """Right-hand sides of the full-coverage identities, per row:
    m1[i]   = sum_k W^M_{i,k}                   (= (M 1)_i by partition of unity)
    mx[i,a] = sum_k W^M_{i,k} x^M_{k,a}         (= (M g^a)_i by linear reproduction)
    kx[i,a] = sum_k W^{K,a}_{i,k}               (= (K g^a)_i; its x-derivative is 1)
    computed directly from the rules and c (no basis tables involved)."""
    ns = dims(n, d)
    tabs = [tables_1d(p, na, mode) for na in ns]
    Ns = [na + p for na in ns]
    m1 = np.zeros(len(rows))
    mx = np.zeros((len(rows), d))
    kx = np.zeros((len(rows), d))
    for ri, row in enumerate(rows):
        idx = decode(int(row), Ns, d)
        R = [tabs[a][i] for a, i in enumerate(idx)]
        X = np.meshgrid(*[r.xM for r in R], indexing="ij")
        W = coeff.evaluate(desc, n, X, grid, plane0)
        for a in range(d):
            shape = [1] * d
            shape[a] = -1
            W = W * R[a].wM.reshape(shape)
        m1[ri] = W.sum()
        for a in range(d):
            mx[ri, a] = (W * X[a]).sum()
            Xa = np.meshgrid(*[R[b].xK if b == a else R[b].xM for b in range(d)], indexing="ij")
            Wa = coeff.evaluate(desc, n, Xa, grid, plane0)
            for b in range(d):
                shape = [1] * d
                shape[b] = -1
                Wa = Wa * (R[b].wK if b == a else R[b].wM).reshape(shape)
            kx[ri, a] = Wa.sum()
    return m1, mx, kx


def greville(p, n):
    """Greville abscissae g_j = (t_{j+1} + ... + t_{j+p}) / p: sum_j g_j B_j(x) = x."""
    t = spline.open_uniform_knots(p, n)
    return np.array([t[j + 1:j + p + 1].mean() for j in range(n + p)])


def ell_columns(p, n, d, row):
    """Global column index of every ELL slot of ``row`` (-1 where out of range)."""
    Ns = [na + p for na in dims(n, d)]
    s = 2 * p + 1
    idx = decode(int(row), Ns, d)
    cols = np.full(s ** d, -1, dtype=np.int64)
    for slot in range(s ** d):
        rem, col, stride, ok = slot, 0, 1, True
        for a in range(d):
            o = rem % s - p
            rem //= s
            j = idx[a] + o
            if not 0 <= j < Ns[a]:
                ok = False
            col += j * stride
            stride *= Ns[a]
        if ok:
            cols[slot] = col
    return cols
