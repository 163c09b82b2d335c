"""Weighted Gaussian quadrature rules -- ORACLE (test infrastructure only).

Convention (eq:GaussQuadW / eq:GaussQuadSys and eq:GaussQuadSysStiff):
the rule for the weight W = B_j (mass) or W = B'_j (stiffness) is

    int_{supp B_j} f(x) W(x) dx  ~=  sum_k omega_k f(tau_k) W(tau_k),

and it is exact for every f = B_i (mass) or f = B'_i (stiffness) with i in the
interacting set {j-p .. j+p}.  The *effective
weight* of node k is omega_k W(tau_k).

Everything here is in unit element spacing ("cardinal").  Nodes are
measured from the left end of supp B_j.  ``rules_1d`` maps the unit rules onto a
mesh of spacing h = 1/n (nodes h*(e0 + tau), omega -> h*omega) for each of the
N = n + p basis functions of one direction.

Interior rules follow the paper step by step:
  * p=2 mass   : symmetry + tau_2 = 3/2, the 3x3 system eq:QuadraticQuadrature
  * p=3 mass   : symmetry, the 4x4 system eq:CubicQuadrature with the brackets
                 tau_1 in (0,1), tau_2 in (1,2) of P:326, solved by Newton
  * p=2 stiff  : symmetry + tau_2 = 3/2, eq:QuadraticQuadratureStiff;
                 omega_2 multiplies B'_j(3/2) = 0 and is free: the printed 8/9 is kept
                 (reading R2); lines 1-2 are solved with true signs (R3)
  * p=3 stiff  : omega_1 = 1, tau_1 the smaller root in (0,1) of the quartic
                 eq:CubicStiffTau1W, then lines 2 and 4 of
                 eq:CubicQuadratureStiff for (tau_2, omega_2) (R3, R8)
Boundary rows (remark P:438-440) follow DESIGN.md reading R1.
"""
import itertools

import numpy as np

from . import quadrature, spline


class Rule:
    """A unit-spacing weighted rule: nodes ``tau`` (from the left end of the
    weight's support), weights ``omega`` in the paper's convention."""

    def __init__(self, kind, p, cls, tau, omega, residual, note=""):
        self.kind, self.p, self.cls = kind, p, cls
        self.tau = np.asarray(tau, dtype=np.float64)
        self.omega = np.asarray(omega, dtype=np.float64)
        self.residual = float(residual)
        self.note = note

    @property
    def m(self):
        return len(self.tau)

    def __repr__(self):
        return f"Rule({self.kind}, p={self.p}, {self.cls}, tau={self.tau}, omega={self.omega}, res={self.residual:.2e})"


# ----------------------------------------------------------------------------------------
# reference (unit spacing) spline space used to derive the rules
# ----------------------------------------------------------------------------------------
def reference_knots(p):
    """Open knot vector with unit spacing and n_ref = 4p+2 elements (enough for a
    weight whose 2p+1 interacting functions are all cardinal)."""
    n_ref = 4 * p + 2
    return spline.open_uniform_knots(p, n_ref, length=float(n_ref)), n_ref


def interior_index(p):
    """Index of a fully cardinal weight in the reference space: j = 2p, supp = [p, 2p+1]."""
    return 2 * p


def _system(t, p, j, order, rows):
    """Residual and Jacobian blocks of the exactness system for weight B_j^{(order)}."""
    mu = quadrature.moments(t, p, j, "mass" if order == 0 else "stiffness", rows)
    lo, _ = spline.support(t, j, p)

    def evaluate(tau_rel, omega):
        x = lo + np.asarray(tau_rel, dtype=np.float64)
        W = spline.deriv(t, j, p, x, order)
        dW = spline.deriv(t, j, p, x, order + 1)
        F = np.array([spline.deriv(t, i, p, x, order) for i in rows])        # [rows, k]
        dF = np.array([spline.deriv(t, i, p, x, order + 1) for i in rows])
        r = F @ (omega * W) - mu
        J_tau = omega[None, :] * (dF * W[None, :] + F * dW[None, :])
        J_omega = F * W[None, :]
        return r, J_tau, J_omega

    return evaluate


class _Param:
    """Linear parametrisation tau = Tm u + tb, omega = Wm u + wb."""

    def __init__(self, Tm, tb, Wm, wb):
        self.Tm, self.tb, self.Wm, self.wb = (np.asarray(a, dtype=np.float64) for a in (Tm, tb, Wm, wb))

    def tau(self, u):
        return self.Tm @ u + self.tb

    def omega(self, u):
        return self.Wm @ u + self.wb


def _newton(evaluate, param, u0, brackets, iters=40, tol=2e-16):
    """Damped Newton with step halving and projection of each free node into its
    bracket (the "element brackets" of P:326).  Returns (u, max|r|)."""
    u = np.array(u0, dtype=np.float64)

    def project(v):
        v = v.copy()
        for idx, (a, b) in brackets.items():
            eps = 1e-12 * (b - a)
            v[idx] = min(max(v[idx], a + eps), b - eps)
        return v

    def res(v):
        r, Jt, Jw = evaluate(param.tau(v), param.omega(v))
        return r, Jt @ param.Tm + Jw @ param.Wm

    u = project(u)
    r, J = res(u)
    nr = np.max(np.abs(r))
    for _ in range(iters):
        if nr <= tol:
            break
        try:
            du = np.linalg.lstsq(J, r, rcond=None)[0]
        except np.linalg.LinAlgError:
            break
        lam, accepted = 1.0, False
        while lam > 1e-6:
            v = project(u - lam * du)
            rv, Jv = res(v)
            nv = np.max(np.abs(rv))
            if np.isfinite(nv) and nv < nr:
                u, r, J, nr, accepted = v, rv, Jv, nv, True
                break
            lam *= 0.5
        if not accepted:
            break
    return u, nr


def _polish(t, p, j, order, rows, param, u, dps=40):
    """Refine a converged fp64 root of the same system in mpmath (``dps`` digits) and round
    it once, so that the rule is correctly rounded rather than accurate to the fp64 residual
    floor times the system's condition number (R14)."""
    import mpmath as mp
    with mp.workdps(dps):
        tk = [mp.mpf(float(v)) for v in t]
        lo = tk[j]
        hi = tk[j + p + 1]

        def moment(i):
            total = mp.mpf(0)
            for s in range(len(tk) - 1):
                a, b = tk[s], tk[s + 1]
                if b > a and a >= lo and b <= hi:
                    total += mp.quad(lambda x: spline.deriv_scalar(tk, i, p, x, order) *
                                     spline.deriv_scalar(tk, j, p, x, order), [a, b])
            return total

        mu = [moment(i) for i in rows]
        Tm = [[mp.mpf(float(v)) for v in r] for r in param.Tm]
        Wm = [[mp.mpf(float(v)) for v in r] for r in param.Wm]
        tb = [mp.mpf(float(v)) for v in param.tb]
        wb = [mp.mpf(float(v)) for v in param.wb]

        def F(*uu):
            tau = [sum(Tm[k][q] * uu[q] for q in range(len(uu))) + tb[k] for k in range(len(tb))]
            om = [sum(Wm[k][q] * uu[q] for q in range(len(uu))) + wb[k] for k in range(len(wb))]
            res = []
            for ri, i in enumerate(rows):
                acc = mp.mpf(0)
                for k in range(len(tau)):
                    x = lo + tau[k]
                    acc += om[k] * spline.deriv_scalar(tk, i, p, x, order) * spline.deriv_scalar(tk, j, p, x, order)
                res.append(acc - mu[ri])
            return res

        x0 = [mp.mpf(float(v)) for v in u]
        sol = mp.findroot(F, x0, solver="mdnewton", tol=mp.mpf(10) ** (-2 * dps + 12), maxsteps=60)
        sol = [sol] if len(u) == 1 else list(sol)
        return np.array([float(v) for v in sol])


def _polished(t, p, j, order, rows, param, u):
    v = _polish(t, p, j, order, rows, param, u)
    if np.max(np.abs(v - u)) > 1e-12:
        raise RuntimeError("high-precision refinement moved the root: %s -> %s" % (u, v))
    return v


def full_residual(rule, t=None):
    """max_i |sum_k omega_k F_i(tau_k) W(tau_k) - mu_i| over the FULL interacting set."""
    p = rule.p
    if t is None:
        t, _ = reference_knots(p)
    order = 0 if rule.kind == "mass" else 1
    if rule.cls == "interior":
        j = interior_index(p)
    else:
        j = rule.cls[1]
    rows = [i for i in range(j - p, j + p + 1) if 0 <= i < len(t) - p - 1]
    ev = _system(t, p, j, order, rows)
    r, _, _ = ev(rule.tau, rule.omega)
    return float(np.max(np.abs(r)))


# ----------------------------------------------------------------------------------------
# interior rules (Sec. 3.1, 3.2)
# ----------------------------------------------------------------------------------------
def interior_mass_p2():
    """eq:QuadraticQuadrature: tau = (tau1, 3/2, 3 - tau1), omega = (w1, w2, w1);
    unknowns (tau1, w1, w2); the three equations are offsets i - j = -2, -1, 0."""
    p = 2
    t, _ = reference_knots(p)
    j = interior_index(p)
    ev = _system(t, p, j, 0, [j - 2, j - 1, j])
    param = _Param(Tm=[[1, 0, 0], [0, 0, 0], [-1, 0, 0]], tb=[0, 1.5, 3.0],
                   Wm=[[0, 1, 0], [0, 0, 1], [0, 1, 0]], wb=[0, 0, 0])
    u, nr = _newton(ev, param, [0.5, 1.0, 1.0], {0: (0.0, 1.0)})
    u = _polished(t, p, j, 0, [j - 2, j - 1, j], param, u)
    rule = Rule("mass", p, "interior", param.tau(u), param.omega(u), 0.0, "eq:WQquadratic")
    rule.residual = full_residual(rule)
    return rule


def interior_mass_p3(starts=None):
    """eq:CubicQuadrature: symmetric 4-node rule, unknowns (tau1, tau2, w1, w2),
    brackets tau1 in (0,1), tau2 in (1,2), offsets -3..0.  Deterministic
    multi-start from element midpoints +- {0, 0.2, 0.35}; first admissible root wins."""
    p = 3
    t, _ = reference_knots(p)
    j = interior_index(p)
    ev = _system(t, p, j, 0, [j - 3, j - 2, j - 1, j])
    param = _Param(Tm=[[1, 0, 0, 0], [0, 1, 0, 0], [0, -1, 0, 0], [-1, 0, 0, 0]], tb=[0, 0, 4, 4],
                   Wm=[[0, 0, 1, 0], [0, 0, 0, 1], [0, 0, 0, 1], [0, 0, 1, 0]], wb=[0, 0, 0, 0])
    if starts is None:
        offs = [0.0, 0.2, -0.2, 0.35, -0.35]
        starts = [[0.5 + a, 1.5 + b, 1.0, 1.0] for a in offs for b in offs]
    for s in starts:
        u, nr = _newton(ev, param, s, {0: (0.0, 1.0), 1: (1.0, 2.0)})
        tau, om = param.tau(u), param.omega(u)
        if nr < 1e-13 and 0 < tau[0] < 1 and 1 < tau[1] < 2 and np.all(om > 0):
            u = _polished(t, p, j, 0, [j - 3, j - 2, j - 1, j], param, u)
            tau, om = param.tau(u), param.omega(u)
            rule = Rule("mass", p, "interior", tau, om, 0.0, "eq:WQcubic")
            rule.residual = full_residual(rule)
            return rule
    raise RuntimeError("p=3 interior mass rule: no admissible root")


def interior_stiff_p2(omega2=8.0 / 9.0):
    """eq:QuadraticQuadratureStiff: tau = (tau1, 3/2, 3 - tau1), omega = (w1, w2, w1).
    B'_j(3/2) = 0 so w2 is free (reading R2; the printed 8/9 is kept).  Unknowns (tau1, w1)
    from the offsets -2, -1 with true signs (reading R3); offset 0 is checked by the residual."""
    p = 2
    t, _ = reference_knots(p)
    j = interior_index(p)
    ev = _system(t, p, j, 1, [j - 2, j - 1])
    param = _Param(Tm=[[1, 0], [0, 0], [-1, 0]], tb=[0, 1.5, 3.0],
                   Wm=[[0, 1], [0, 0], [0, 1]], wb=[0, omega2, 0])
    u, nr = _newton(ev, param, [0.5, 1.0], {0: (0.0, 1.0)})
    u = _polished(t, p, j, 1, [j - 2, j - 1], param, u)
    rule = Rule("stiffness", p, "interior", param.tau(u), param.omega(u), 0.0, "eq:WQquadraticStiff")
    rule.residual = full_residual(rule)
    return rule


def cubic_stiff_tau1(omega1=1.0):
    """Roots of eq:CubicStiffTau1W 30 w1 x^4 - 60 w1 x^3 + 30 w1 x^2 - 1 = 0 in (0,1);
    the smaller one is taken."""
    roots = np.roots([30.0 * omega1, -60.0 * omega1, 30.0 * omega1, 0.0, -1.0])
    real = sorted(float(r.real) for r in roots if abs(r.imag) < 1e-12 and 0.0 < r.real < 1.0)
    if not real:
        raise ValueError("eq:CubicStiffTau1W has no root in (0,1) for omega1=%g" % omega1)
    return real


def interior_stiff_p3(omega1=1.0):
    """eq:CubicQuadratureStiff: omega1 fixed (=1), tau1 the smaller root of
    eq:CubicStiffTau1W, then lines 2 and 4 (offsets -2 and 0) for (tau2, omega2) with
    tau2 in (1,2); line 3 (offset -1, corrected per reading R3) is checked by the residual."""
    p = 3
    t, _ = reference_knots(p)
    j = interior_index(p)
    tau1 = cubic_stiff_tau1(omega1)[0]
    ev = _system(t, p, j, 1, [j - 2, j])
    param = _Param(Tm=[[0, 0], [1, 0], [-1, 0], [0, 0]], tb=[tau1, 0, 4, 4 - tau1],
                   Wm=[[0, 0], [0, 1], [0, 1], [0, 0]], wb=[omega1, 0, 0, omega1])
    offs = [0.0, 0.2, -0.2, 0.35, -0.35]
    for a in offs:
        u, nr = _newton(ev, param, [1.5 + a, 1.0], {0: (1.0, 2.0)})
        tau, om = param.tau(u), param.omega(u)
        if nr < 1e-13 and 1 < tau[1] < 2 and np.all(om > 0):
            # refine tau1 (line 1 = the quartic), tau2, omega2 together (lines 1, 2, 4)
            pfull = _Param(Tm=[[1, 0, 0], [0, 1, 0], [0, -1, 0], [-1, 0, 0]], tb=[0, 0, 4, 4],
                           Wm=[[0, 0, 0], [0, 0, 1], [0, 0, 1], [0, 0, 0]], wb=[omega1, 0, 0, omega1])
            v = _polished(t, p, j, 1, [j - 3, j - 2, j], pfull, np.array([tau1, u[0], u[1]]))
            tau, om = pfull.tau(v), pfull.omega(v)
            rule = Rule("stiffness", p, "interior", tau, om, 0.0, "eq:WQcubicStiff")
            rule.residual = full_residual(rule)
            return rule
    raise RuntimeError("p=3 interior stiffness rule: no admissible completion")


# ----------------------------------------------------------------------------------------
# boundary rows (remark P:438-440, reading R1)
# ----------------------------------------------------------------------------------------
GL_FALLBACK = {("stiffness", 2, 1), ("stiffness", 3, 1)}   # reading R1: no admissible minimal rule


def boundary_dimension(kind, p, j):
    """Number of independent exactness constraints for the left boundary weight j:
    mass D = p+j+1 (restricted spline space), stiffness D = p+j (its derivatives)."""
    return p + j + 1 if kind == "mass" else p + j


def gl_rule(kind, p, j):
    """Standard Gauss rule on the support (the paper's alternative): (p+1)-point
    Gauss-Legendre on every element of [0, j+1]; omega are the GL weights (the rule then
    integrates f*W exactly for every polynomial f*W of degree <= 2p+1 per element)."""
    import mpmath as mp
    tau, om = [], []
    m = p + 1
    for e in range(j + 1):
        x, w = quadrature.gauss_legendre(m, float(e), float(e + 1))
        # refine each node as a root of P_m(2x - 1) in 40 digits; w = 1/((1-s^2) P_m'(s)^2)
        with mp.workdps(40):
            for xi in x:
                s = mp.findroot(lambda z: mp.legendre(m, z), mp.mpf(2 * (float(xi) - e) - 1))
                dP = mp.diff(lambda z: mp.legendre(m, z), s)
                tau.append(float(e + (s + 1) / 2))
                om.append(float(1 / ((1 - s * s) * dP * dP)))
    rule = Rule(kind, p, ("left", j), tau, om, 0.0, "GL(p+1) per element")
    rule.residual = full_residual(rule)
    return rule


def boundary_gauss(kind, p, j, grid_points=7):
    """Minimal Gaussian rule for the left boundary weight j (reading R1):
    m = ceil(D/2) nodes; when D is odd the last node is fixed at j + 1/2 (the midpoint
    of the last element of the support, as the paper fixes tau_2 = 3/2 at P:262).
    Deterministic multi-start over an increasing grid of nodes in (0, j+1); every
    admissible root (nodes strictly inside, increasing, positive weights) is collected
    and must be unique."""
    order = 0 if kind == "mass" else 1
    t, _ = reference_knots(p)
    D = boundary_dimension(kind, p, j)
    m = (D + 1) // 2
    fixed = (D % 2 == 1)
    nfree = m - 1 if fixed else m
    rows = list(range(0, j + p + 1))
    if kind == "stiffness":
        rows = rows[:-1]          # sum_i B'_i = 0 on [0, j+1]: the last equation is implied
    ev = _system(t, p, j, order, rows)
    L = float(j + 1)
    nu = nfree + m
    Tm = np.zeros((m, nu))
    tb = np.zeros(m)
    for k in range(nfree):
        Tm[k, k] = 1.0
    if fixed:
        tb[m - 1] = j + 0.5
    Wm = np.zeros((m, nu))
    for k in range(m):
        Wm[k, nfree + k] = 1.0
    param = _Param(Tm, tb, Wm, np.zeros(m))
    grid = np.linspace(0.04, 0.96, grid_points) * L
    roots = []
    for combo in itertools.combinations(grid, nfree):
        if fixed and max(combo, default=0.0) >= j + 0.5:
            continue
        u0 = np.concatenate([np.array(combo), np.full(m, 1.0 / m)])
        u, nr = _newton(ev, param, u0, {k: (0.0, L) for k in range(nfree)})
        tau, om = param.tau(u), param.omega(u)
        if nr > 1e-13:
            continue
        if not (np.all(tau > 1e-9) and np.all(tau < L - 1e-9) and np.all(np.diff(tau) > 1e-9) and np.all(om > 0)):
            continue
        if not any(np.max(np.abs(tau - r[0])) < 1e-8 for r in roots):
            roots.append((tau, om))
    if not roots:
        return None, 0
    tau, om = roots[0]
    u = np.concatenate([tau[:nfree], om])
    u = _polished(t, p, j, order, rows, param, u)
    tau, om = param.tau(u), param.omega(u)
    rule = Rule(kind, p, ("left", j), tau, om, 0.0, "boundary Gauss (R1)")
    rule.residual = full_residual(rule)
    return rule, len(roots)


def boundary_rule(kind, p, j, mode="gauss"):
    if mode == "gl" or (kind, p, j) in GL_FALLBACK:
        return gl_rule(kind, p, j)
    rule, count = boundary_gauss(kind, p, j)
    if rule is None:
        raise RuntimeError(f"no admissible boundary rule for {kind} p={p} j={j}")
    if count != 1:
        raise RuntimeError(f"{count} admissible boundary rules for {kind} p={p} j={j}")
    return rule


_CACHE = {}


def class_rules(p, mode="gauss"):
    """All unit-spacing rules for degree p: {'mass'|'stiffness': {'interior': Rule, j: Rule}}."""
    key = (p, mode)
    if key in _CACHE:
        return _CACHE[key]
    if p == 2:
        interior = {"mass": interior_mass_p2(), "stiffness": interior_stiff_p2()}
    elif p == 3:
        interior = {"mass": interior_mass_p3(), "stiffness": interior_stiff_p3()}
    else:
        raise ValueError("the paper derives rules for p = 2, 3 only")
    out = {}
    for kind in ("mass", "stiffness"):
        out[kind] = {"interior": interior[kind]}
        for j in range(p):
            out[kind][j] = boundary_rule(kind, p, j, mode)
    _CACHE[key] = out
    return out


# ----------------------------------------------------------------------------------------
# rules on a mesh of n uniform elements (h = 1/n)
# ----------------------------------------------------------------------------------------
class Rule1D:
    """The rule of 1D row r on the physical mesh: nodes x (ascending), omega (physical),
    effective weights w = omega * W(x) with W = B_r (mass) or B'_r (stiffness, physical
    derivative)."""

    def __init__(self, x, omega, w):
        self.x, self.omega, self.w = x, omega, w


def rules_1d(p, n, kind, mode="gauss"):
    """Per-row rules for the N = n+p basis functions of one direction (h = 1/n).

    r < p          : left boundary class j = r   (nodes h*tau)
    p <= r <= n-1  : interior rule              (nodes h*(r-p+tau)), P:248 supp = [xi_r, xi_{r+p+1}]
    r >= n         : right boundary class j = N-1-r, mirrored x -> 1 - x (reading R1)
    omega scales by h (d x = h d tau); derivative values are physical (1/h per derivative).
    """
    if n < p:
        raise ValueError("n_elems must be >= p")
    cr = class_rules(p, mode)[kind]
    t = spline.open_uniform_knots(p, n)
    h = 1.0 / n
    N = n + p
    order = 0 if kind == "mass" else 1
    out = []
    for r in range(N):
        if r < p:
            rule = cr[r]
            x = h * rule.tau
            om = h * rule.omega
        elif r >= n:
            rule = cr[N - 1 - r]
            x = (1.0 - h * rule.tau)[::-1]
            om = (h * rule.omega)[::-1]
        else:
            rule = cr["interior"]
            x = h * ((r - p) + rule.tau)
            om = h * rule.omega
        W = spline.deriv(t, r, p, x, order)
        out.append(Rule1D(np.array(x), np.array(om), om * W))
    return out


