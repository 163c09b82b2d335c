"""Counter-based generators for the synthetic coefficient fields.

sm(z) is the splitmix64 finaliser (mix only, no increment); u(z) = (z >> 11) * 2^-53.
"""
import math

import numpy as np

SEED = 171001048
GAMMA = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
# sqrt((C(16,8) / 2^16)^3): standard deviation of three binomial-8 passes applied to
# unit white noise (c.4 step 3 quotes it rounded as 0.087026).
GRID_NORM = math.sqrt((12870.0 / 65536.0) ** 3)
BINOMIAL8 = np.array([1, 8, 28, 56, 70, 56, 28, 8, 1], dtype=np.float64) / 256.0


def splitmix64(z):
    """splitmix64 finaliser on uint64 (scalar int or numpy array)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(M2)
        z = z ^ (z >> np.uint64(31))
    return z


def u53(z):
    """Uniform double in [0, 1) from the top 53 bits."""
    return (np.asarray(z, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _stream(seed, t):
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + np.asarray(t, dtype=np.uint64) * np.uint64(GAMMA)
    return u53(splitmix64(z))


def fourier_modes(seed=SEED, n_modes=8, amp=0.3, dim=2):
    """FOURIER_LOGN parameters: rows (a_m, kx_m, ky_m, kz_m, theta_m), m = 1..n_modes.

    d_t = u(sm(seed + t*GAMMA)); k^x_m = m; k^y = Fisher-Yates permutation of 1..M from
    d_0..d_{M-2} (j = floor(d*(i+1)), i = M-1..1); theta_m = 2 pi d_{M-2+m};
    z_m = sqrt(-2 ln(1-d_{2M-3+2m})) cos(2 pi d_{2M-2+2m}); a = amp * z * sqrt(M)/|z|.
    (For M = 8 these are exactly the indices of c.4.)  kz = 0 (the C3 field is 2D).
    """
    M = n_modes
    d = _stream(seed, np.arange(4 * M, dtype=np.uint64))
    perm = list(range(1, M + 1))
    t = 0
    for i in range(M - 1, 0, -1):
        j = int(math.floor(d[t] * (i + 1)))
        t += 1
        perm[i], perm[j] = perm[j], perm[i]
    theta = np.array([2.0 * math.pi * d[M - 2 + m] for m in range(1, M + 1)])
    z = np.array([math.sqrt(-2.0 * math.log(1.0 - d[2 * M - 3 + 2 * m])) * math.cos(2.0 * math.pi * d[2 * M - 2 + 2 * m])
                  for m in range(1, M + 1)])
    a = amp * z * math.sqrt(M) / np.linalg.norm(z)
    modes = np.zeros((M, 5))
    modes[:, 0] = a
    modes[:, 1] = np.arange(1, M + 1)
    modes[:, 2] = perm if dim >= 2 else 0
    modes[:, 3] = 0.0
    modes[:, 4] = theta
    return modes


def _white(seed, n, idx3):
    """g0 at extended vertices given as (a, b, c) index arrays in [-4, n_a+4]; n = elements per
    direction (int or (n_x, n_y[, n_z])): key = ((c+4) ext_y + (b+4)) ext_x + (a+4), ext = n + 9
    (for equal counts the key of SURVEY §8(c) c.4)."""
    a, b, c = idx3
    nx, ny = (n, n) if np.ndim(n) == 0 else (int(n[0]), int(n[1]))
    key = ((c + 4) * (ny + 9) + (b + 4)) * (nx + 9) + (a + 4)
    key = key.astype(np.uint64)
    with np.errstate(over="ignore"):
        k2 = key * np.uint64(2)
        u1 = u53(splitmix64(np.uint64(seed) ^ k2))
        u2 = u53(splitmix64(np.uint64(seed) ^ (k2 + np.uint64(1))))
    return np.sqrt(-2.0 * np.log(1.0 - u1)) * np.cos(2.0 * math.pi * u2)


def lognormal_grid(n, seed=SEED, sigma=0.5, dim=3, plane0=0, planes=None):
    """Smoothed lognormal vertex field c = exp(sigma * g) on vertices 0..n (c.4).

    dim=3: returns [planes, n+1, n+1] for vertex planes c in [plane0, plane0+planes),
    indexed [c][b][a] (x fastest).  dim=2: returns [planes, n+1] for rows b (key uses c=0).
    dim=1: returns [n+1] (keys use b=c=0).
    Every value is a function of its global key only, so any slab equals the same slab
    of the global field.  n may give the element count per direction (x, y[, z]): vertex
    planes then hold (n_y+1) x (n_x+1) values and the slowest axis has n_dim + 1 planes.
    """
    ns = [int(n)] * dim if np.ndim(n) == 0 else [int(v) for v in n][:dim]
    n = (ns[0], ns[1] if dim >= 2 else ns[0])         # the key strides (x, y)
    nv = ns[dim - 1] + 1
    if planes is None:
        planes = nv - plane0
    ax = np.arange(-4, ns[0] + 1 + 4, dtype=np.int64)
    if dim == 3:
        cz = np.arange(plane0 - 4, plane0 + planes + 4, dtype=np.int64)
        ay = np.arange(-4, ns[1] + 1 + 4, dtype=np.int64)
        C, B, A = np.meshgrid(cz, ay, ax, indexing="ij")
        g = _white(seed, n, (A, B, C))
        for axis in (2, 1, 0):
            g = _valid_filter(g, axis)
    elif dim == 2:
        by = np.arange(plane0 - 4, plane0 + planes + 4, dtype=np.int64)
        B, A = np.meshgrid(by, ax, indexing="ij")
        g = _white(seed, n, (A, B, np.zeros_like(A)))
        for axis in (1, 0):
            g = _valid_filter(g, axis)
    else:
        g = _white(seed, n, (ax, np.zeros_like(ax), np.zeros_like(ax)))
        g = _valid_filter(g, 0)
    norm = GRID_NORM if dim == 3 else math.sqrt((12870.0 / 65536.0) ** dim)
    return np.exp(sigma * (g / norm))


def _valid_filter(g, axis):
    """'valid' binomial-8 filter along one axis (shrinks that axis by 8)."""
    L = g.shape[axis] - 8
    out = np.zeros(g.shape[:axis] + (L,) + g.shape[axis + 1:])
    for tap in range(9):
        sl = [slice(None)] * g.ndim
        sl[axis] = slice(tap, tap + L)
        out += BINOMIAL8[tap] * g[tuple(sl)]
    return out
