"""Pins for oracle/coeff.py (no GPU): the coefficient fields every parity case samples.

Each check is independent of the oracle's own arithmetic:

* FOURIER_LOGN (C3, DESIGN R13): the parameters (a_m, k_m, theta_m) are
  rebuilt here from the raw splitmix64 stream with Python integers (not through
  ``inputs.fourier_modes``), and c = exp(sum_m a_m cos(2 pi (k.x) + theta_m)) is evaluated in
  30-digit mpmath at seeded points.  A second pin needs no re-evaluation at all: with distinct
  integer wavevectors the modes are orthogonal on a cell-centred grid, so mean(log c) = 0 and
  mean((log c)^2) = sum a_m^2 / 2 = 0.36 exactly (std 0.6, c.4).
* TRIG_SEP (C2, C4): c0 + amp prod_a trig(2 pi k_a x_a) in mpmath.
* GRID (C5, R6): the multilinear interpolant reproduces every multilinear polynomial exactly
  (x, y, z, xy, xz, yz, xyz and their sums), at any point and on any slab of vertex planes
  (plane0 != 0): a wrong fraction, a wrong axis or a wrong plane offset breaks it.
"""
import math

import mpmath
import numpy as np
import pytest

import inputs
from oracle import coeff

mpmath.mp.dps = 30
MASK = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def sm(z):
    """splitmix64 finaliser (Steele, Lea, Flood 2014) on Python ints."""
    z &= MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def u(z):
    return mpmath.mpf(z >> 11) / mpmath.mpf(2) ** 53


def modes_from_stream(seed, M=8, amp=0.3):
    """c.4 FOURIER_LOGN parameters from d_t = u(sm(seed + t GAMMA)), in mpmath."""
    d = [u(sm(seed + t * GAMMA)) for t in range(4 * M)]
    perm = list(range(1, M + 1))
    for t, i in enumerate(range(M - 1, 0, -1)):        # Fisher-Yates with d_0 .. d_{M-2}
        j = int(mpmath.floor(d[t] * (i + 1)))
        perm[i], perm[j] = perm[j], perm[i]
    theta = [2 * mpmath.pi * d[M - 2 + m] for m in range(1, M + 1)]
    z = [mpmath.sqrt(-2 * mpmath.log(1 - d[2 * M - 3 + 2 * m])) * mpmath.cos(2 * mpmath.pi * d[2 * M - 2 + 2 * m])
         for m in range(1, M + 1)]
    nz = mpmath.sqrt(sum(v * v for v in z))
    a = [amp * v * mpmath.sqrt(M) / nz for v in z]
    return [(a[m], m + 1, perm[m], theta[m]) for m in range(M)]


def c_fourier_mp(modes, pt):
    s = mpmath.mpf(0)
    for a, kx, ky, th in modes:
        ph = kx * mpmath.mpf(pt[0])
        if len(pt) > 1:
            ph += ky * mpmath.mpf(pt[1])
        s += a * mpmath.cos(2 * mpmath.pi * ph + th)
    return mpmath.exp(s)


@pytest.mark.parametrize("seed", [inputs.SEED, 3, 11])
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_fourier_logn_matches_mpmath_from_raw_stream(seed, dim):
    modes = modes_from_stream(seed)
    desc = inputs.coefficient({"kind": "fourier_logn", "seed": seed, "n_modes": 8, "amp": 0.3}, dim)
    rng = np.random.default_rng(seed)
    pts = rng.random((50, dim))
    pts[:4] = [[0.0] * dim, [1.0] * dim, [0.5] * dim, [1.0 / 3] * dim]
    got = coeff.evaluate(desc, 8, [pts[:, a] for a in range(dim)])
    # the C3 field is 2D: in 3D it does not depend on z, in 1D it is the y = 0 section
    ref = np.array([float(c_fourier_mp(modes, pt[:2])) for pt in pts])
    assert np.max(np.abs(got - ref) / ref) < 1e-13


def test_fourier_logn_c3_statistics_exact():
    """Distinct integer wavevectors (m, pi(m)), |k| <= 8: on a 32 x 32 cell-centred grid the
    cosines are orthogonal, so mean(log c) = 0 and mean((log c)^2) = sum a^2 / 2 = 0.3^2 8 / 2."""
    desc = inputs.coefficient(inputs.config("C3")["coeff"], 2)
    L = 32
    ax = (np.arange(L) + 0.5) / L
    Y, X = np.meshgrid(ax, ax, indexing="ij")
    lc = np.log(coeff.evaluate(desc, L, [X, Y]))
    assert abs(lc.mean()) < 1e-14
    assert abs((lc ** 2).mean() - 0.36) < 1e-13
    ks = {(m[1], m[2]) for m in desc["modes"]}
    assert len(ks) == 8 and sorted(k[0] for k in ks) == list(range(1, 9)) and sorted(k[1] for k in ks) == list(range(1, 9))


@pytest.mark.parametrize("dim,trig,wave", [(1, ("sin",), (1,)), (2, ("sin", "cos"), (1, 1)),
                                           (3, ("sin", "sin", "sin"), (1, 1, 1)), (3, ("cos", "sin", "cos"), (2, 1, 3))])
def test_trig_sep_matches_mpmath(dim, trig, wave):
    desc = {"kind": "trig_sep", "c0": 1.0, "amp": 0.3, "trig": trig, "wavenum": wave}
    pts = np.random.default_rng(dim).random((40, dim))
    got = coeff.evaluate(desc, 8, [pts[:, a] for a in range(dim)])
    for g, pt in zip(got, pts):
        prod = mpmath.mpf(1)
        for a in range(dim):
            f = mpmath.sin if trig[a] == "sin" else mpmath.cos
            prod *= f(2 * mpmath.pi * wave[a] * mpmath.mpf(pt[a]))
        ref = 1 + mpmath.mpf("0.3") * prod
        assert abs(g - float(ref)) < 4e-16 * 4


MULTILIN = {                      # monomials x^a y^b z^c, a, b, c in {0, 1}
    "1": lambda x, y, z: np.ones_like(x), "x": lambda x, y, z: x, "y": lambda x, y, z: y, "z": lambda x, y, z: z,
    "xy": lambda x, y, z: x * y, "xz": lambda x, y, z: x * z, "yz": lambda x, y, z: y * z,
    "xyz": lambda x, y, z: x * y * z,
}


def _vertex_values(n, f, plane0=0, planes=None, dim=3):
    ax = np.arange(n + 1) / n
    if dim == 3:
        zs = np.arange(plane0, plane0 + (planes or n + 1 - plane0)) / n
        Z, Y, X = np.meshgrid(zs, ax, ax, indexing="ij")
        return f(X, Y, Z)
    ys = np.arange(plane0, plane0 + (planes or n + 1 - plane0)) / n
    Y, X = np.meshgrid(ys, ax, indexing="ij")
    return f(X, Y, np.zeros_like(X))


@pytest.mark.parametrize("name", list(MULTILIN))
@pytest.mark.parametrize("plane0,planes", [(0, None), (3, 4), (6, 3)])
def test_grid_reproduces_multilinear_monomials_3d(name, plane0, planes):
    n = 9
    f = MULTILIN[name]
    grid = _vertex_values(n, f, plane0, planes)
    zlo, zhi = plane0 / n, (plane0 + grid.shape[0] - 1) / n        # the slab's vertex planes
    rng = np.random.default_rng(len(name) + plane0)
    x, y = rng.random(200), rng.random(200)
    z = zlo + (zhi - zlo) * rng.random(200)
    got = coeff.evaluate({"kind": "grid"}, n, [x, y, z], grid=grid, plane0=plane0)
    assert np.max(np.abs(got - f(x, y, z))) < 1e-15 * 4


@pytest.mark.parametrize("plane0,planes", [(0, None), (2, 5)])
def test_grid_reproduces_random_multilinear_2d_and_3d(plane0, planes):
    rng = np.random.default_rng(plane0)
    cf = rng.standard_normal(8)
    f3 = lambda x, y, z: sum(cf[i] * MULTILIN[k](x, y, z) for i, k in enumerate(MULTILIN))  # noqa: E731
    f2 = lambda x, y, z: cf[0] + cf[1] * x + cf[2] * y + cf[3] * x * y  # noqa: E731
    n = 7
    for dim, f in ((3, f3), (2, f2)):
        grid = _vertex_values(n, f, plane0, planes, dim)
        lo, hi = plane0 / n, (plane0 + grid.shape[0] - 1) / n
        pts = [rng.random(300) for _ in range(dim)]
        pts[-1] = lo + (hi - lo) * pts[-1]
        got = coeff.evaluate({"kind": "grid"}, n, pts, grid=grid, plane0=plane0)
        ref = f(*(pts + [np.zeros(300)] * (3 - dim)))
        assert np.max(np.abs(got - ref)) < 1e-14, dim


def test_grid_interpolates_vertex_values_and_is_linear_on_edges():
    """At a vertex the interpolant returns the vertex value; along a cell edge it is the
    linear blend of the two end values (hat functions, R6)."""
    n = 5
    g = inputs.lognormal_grid(n, seed=4, dim=3)
    idx = np.array([[0, 0, 0], [1, 2, 3], [4, 4, 4], [2, 0, 4], [3, 1, 0]])
    # vertex (a, b, c) approached from inside its cell (the cell of a point is floor(x n))
    for a, b, c in idx:
        pts = [np.array([a / n]), np.array([b / n]), np.array([c / n])]
        assert coeff.evaluate({"kind": "grid"}, n, pts, grid=g)[0] == pytest.approx(g[c, b, a], rel=1e-14)
    t = 0.3
    got = coeff.evaluate({"kind": "grid"}, n, [np.array([(2 + t) / n]), np.array([1 / n]), np.array([3 / n])], grid=g)[0]
    assert got == pytest.approx((1 - t) * g[3, 1, 2] + t * g[3, 1, 3], rel=1e-14)
    got = coeff.evaluate({"kind": "grid"}, n, [np.array([2 / n]), np.array([1 / n]), np.array([(3 + t) / n])], grid=g)[0]
    assert got == pytest.approx((1 - t) * g[3, 1, 2] + t * g[4, 1, 2], rel=1e-14)


def test_fourier_phase_wraps_like_the_definition():
    """c is 1-periodic in every coordinate (integer wavevectors): c(x + 1) = c(x)."""
    desc = inputs.coefficient(inputs.config("C3")["coeff"], 2)
    pts = np.random.default_rng(0).random((30, 2))
    a = coeff.evaluate(desc, 8, [pts[:, 0], pts[:, 1]])
    b = coeff.evaluate(desc, 8, [pts[:, 0] + 1.0, pts[:, 1] + 2.0])
    assert np.max(np.abs(a - b) / a) < 1e-13
    assert math.isclose(float(np.log(coeff.evaluate(desc, 8, [np.array([0.0]), np.array([0.0])]))[0]),
                        float(sum(m[0] * math.cos(m[4]) for m in desc["modes"])), rel_tol=1e-13)
