"""Coefficient fields c(x) -- ORACLE (test infrastructure only).

The paper assembles with c == 1.  BASELINE.json's configs multiply the
integrands of both M and K by a coefficient c (reading R4); each row
samples c at its own quadrature nodes.  Kinds (descriptor dicts, inputs/configs.py):

  const        c = c0
  trig_sep     c = c0 + amp * prod_a trig_a(2 pi k_a x_a)            (C2, C4; reading R13)
  fourier_logn c = exp(sum_m a_m cos(2 pi (kx x + ky y + kz z) + theta_m))   (C3; R13)
  grid         multilinear interpolation of vertex values, vertex (a,b,c) at (a,b,c)/n  (C5; R6)
"""
import math

import numpy as np


def evaluate(desc, n, pts, grid=None, plane0=0):
    """c at points ``pts`` = list of d coordinate arrays (same shape); n = elements per
    direction (int, or one per direction: the GRID vertex spacing is 1/n_a)."""
    kind = desc["kind"]
    d = len(pts)
    if kind == "const":
        return np.full(np.shape(pts[0]), float(desc["c0"]))
    if kind == "trig_sep":
        prod = np.ones(np.shape(pts[0]))
        for a in range(d):
            f = np.sin if desc["trig"][a] == "sin" else np.cos
            prod = prod * f(2.0 * math.pi * desc["wavenum"][a] * pts[a])
        return desc["c0"] + desc["amp"] * prod
    if kind == "fourier_logn":
        # Evaluated in x87 extended precision (64-bit mantissa) and rounded once: the phase
        # 2 pi (k . x) reaches ~100, where a double-precision phase would carry ~1e-14
        # absolute error and make the oracle's own c wrong beyond the parity tolerance.
        ld = np.longdouble
        two_pi = ld(2) * ld("3.14159265358979323846264338327950288")
        s = np.zeros(np.shape(pts[0]), dtype=ld)
        for a_m, kx, ky, kz, th in desc["modes"]:
            arg = ld(kx) * np.asarray(pts[0], dtype=ld)
            if d > 1:
                arg = arg + ld(ky) * np.asarray(pts[1], dtype=ld)
            if d > 2:
                arg = arg + ld(kz) * np.asarray(pts[2], dtype=ld)
            s = s + ld(a_m) * np.cos(two_pi * arg + ld(th))
        return np.exp(s).astype(np.float64)
    if kind == "grid":
        return _multilinear(grid, n, pts, plane0)
    raise ValueError(kind)


def _multilinear(grid, n, pts, plane0):
    """Vertex field interpolation.  grid is indexed [slowest] ... [x]; its slowest axis
    starts at vertex plane ``plane0``.  Cell = element containing the point; vertex j of
    direction a at j / n_a."""
    d = len(pts)
    ns = [int(n)] * d if np.ndim(n) == 0 else [int(v) for v in n][:d]
    cells, fracs = [], []
    for a in range(d):
        s = np.asarray(pts[a], dtype=np.float64) * ns[a]
        e = np.clip(np.floor(s), 0, ns[a] - 1).astype(np.int64)
        cells.append(e)
        fracs.append(s - e)
    out = np.zeros(np.shape(pts[0]))
    for corner in range(2 ** d):
        bits = [(corner >> a) & 1 for a in range(d)]
        wgt = np.ones(np.shape(pts[0]))
        for a in range(d):
            wgt = wgt * (fracs[a] if bits[a] else 1.0 - fracs[a])
        idx = [cells[a] + bits[a] for a in range(d)]
        idx[d - 1] = idx[d - 1] - plane0          # slowest axis is slab-local
        out = out + wgt * grid[tuple(idx[::-1])]
    return out
