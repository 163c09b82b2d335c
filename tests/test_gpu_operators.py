"""GPU parity of the load vector and the matrix-free product against
the oracle (oracle/operators.py), through the C-ABI (wgq_assemble_load, wgq_apply).

Tolerances as for the matrices (north_star, R12): relative Frobenius <= 1e-12 and
max entrywise relative <= 1e-10; for y = A u the entrywise denominator is floored at the
rounding scale sum_j |A|_ij |u_j| (|A| = the oracle's absolute-value assembly), since a
random u makes y_i a cancelling sum.
"""
import numpy as np
import pytest

import inputs
from oracle import assemble as oasm
from oracle import operators as oops

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from parity import compare  # noqa: E402


def check(g, ref, scale, what):
    compare(g, ref, what, scale, rowwise=False)


def coeff_cases(d):
    return [("const", {"kind": "const", "c0": 1.3}),
            ("trig", {"kind": "trig_sep", "c0": 1.0, "amp": 0.5, "trig": ("sin", "cos", "sin")[:d],
                      "wavenum": (1, 1, 2)[:d]}),
            ("fourier", inputs.coefficient({"kind": "fourier_logn", "seed": inputs.SEED, "n_modes": 8, "amp": 0.3}, d)),
            ("grid", {"kind": "grid", "seed": 4, "sigma": 0.5})]


def coef_obj(desc, n, d):
    from paper_1710_01048_b200 import api
    grid = inputs.lognormal_grid(n, seed=desc["seed"], dim=d) if desc["kind"] == "grid" else None
    gt = torch.from_numpy(np.ascontiguousarray(grid)).cuda() if grid is not None else None
    return api.coefficient(desc, gt, 0), grid


SMALL = [(2, 1, 20), (3, 1, 17), (2, 2, 9), (3, 2, 8), (2, 3, 5), (3, 3, 4), (3, 3, 3)]


@pytest.mark.parametrize("p,d,n", SMALL)
def test_load_vector_all_coefficients(p, d, n):
    from paper_1710_01048_b200 import api, wgq
    rules = wgq.Rules(p, n, d)
    rows = np.arange(rules.n_rows)
    for name, desc in coeff_cases(d):
        c, grid = coef_obj(desc, n, d)
        b = api.assemble_load(rules, c)
        torch.cuda.synchronize()
        ref = oops.load_rows(p, n, d, rows, desc, grid=grid)
        check(b.cpu().numpy(), ref, np.abs(ref), (p, d, n, name))


@pytest.mark.parametrize("p,d,n", SMALL)
def test_apply_all_coefficients(p, d, n):
    from paper_1710_01048_b200 import api, wgq
    rules = wgq.Rules(p, n, d)
    rows = np.arange(rules.n_rows)
    u = np.random.default_rng(p * 100 + d * 10 + n).standard_normal(rules.n_rows)
    ut = torch.from_numpy(u).cuda()
    for name, desc in coeff_cases(d):
        c, grid = coef_obj(desc, n, d)
        y = api.apply(rules, c, ut)
        torch.cuda.synchronize()
        absA = oasm.assemble_rows(p, n, d, rows, desc, grid=grid, absolute=True)
        for kind in ("mass", "stiffness"):
            ref = oops.apply_rows(p, n, d, rows, desc, u, kind, grid=grid)
            scale = np.array([absA[kind][i][oasm.ell_columns(p, n, d, r) >= 0] @
                              np.abs(u[oasm.ell_columns(p, n, d, r)[oasm.ell_columns(p, n, d, r) >= 0]])
                              for i, r in enumerate(rows)])
            check(y[kind].cpu().numpy(), ref, scale, (p, d, n, name, kind))


def test_apply_slab_matches_full_and_checks_u_range():
    """A z-slab with u holding only its planes +- p gives the full result's rows; too short a
    u is rejected (WGQ_ERANGE)."""
    from paper_1710_01048_b200 import api, wgq
    p, d, n = 3, 3, 6
    rules = wgq.Rules(p, n, d)
    N = rules.N
    u = torch.from_numpy(np.random.default_rng(3).standard_normal(rules.n_rows)).cuda()
    desc = inputs.coefficient({"kind": "fourier_logn", "seed": 2, "n_modes": 8, "amp": 0.3}, d)
    c = api.coefficient(desc)
    full = api.apply(rules, c, u)
    z0, z1 = 3, 6                                         # rows of planes 3..5
    lo, hi = max(0, z0 - p) * N * N, min(N, z1 + p) * N * N
    part = api.apply(rules, c, u[lo:hi], row_begin=z0 * N * N, row_end=z1 * N * N, u_row0=lo)
    torch.cuda.synchronize()
    for k in ("mass", "stiffness"):
        assert torch.equal(part[k], full[k][z0 * N * N:z1 * N * N])
    with pytest.raises(wgq.WgqError):
        api.apply(rules, c, u[lo + N * N:hi], row_begin=z0 * N * N, row_end=z1 * N * N, u_row0=lo + N * N)


def test_load_full_size_c5_sampled_rows():
    """C5's mesh and device-generated grid: every boundary row class plus random rows."""
    from paper_1710_01048_b200 import api, wgq
    cfg = inputs.config("C5")
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    rules = wgq.Rules(p, n, d)
    grid, plane0 = api.make_grid(rules, cfg["coeff"]["seed"], cfg["coeff"]["sigma"], 0, rules.n_rows)
    c = api.coefficient({"kind": "grid"}, grid, plane0)
    b = api.assemble_load(rules, c)
    torch.cuda.synchronize()
    N = rules.N
    rng = np.random.default_rng(5)
    edge = list(range(0, 2 * p + 2)) + list(range(N - 2 * p - 2, N))
    rows = sorted({sum(int(rng.choice(edge) if rng.random() < 0.5 else rng.integers(0, N)) * N ** a
                       for a in range(d)) for _ in range(300)})
    zs = sorted({r // (N * N) for r in rows})
    host = inputs.lognormal_grid(n, seed=cfg["coeff"]["seed"])
    ref = oops.load_rows(p, n, d, np.array(rows), {"kind": "grid"}, grid=host)
    got = b.cpu().numpy()[rows]
    check(got, ref, np.abs(ref), "C5 load")
    assert len(zs) > 3


@pytest.mark.parametrize("name", ["C5", "C3", "C4", "C2"])
def test_apply_full_size_sampled_rows(name):
    """y = M u, K u at the BASELINE sizes (C5: GRID line kernel, C3: 2D tensor-core kernel, C4 / C2:
    separable kernel) on a
    sample of rows covering every boundary class; u is a seeded random vector."""
    from paper_1710_01048_b200 import api, wgq
    cfg = inputs.config(name)
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    rules = wgq.Rules(p, n, d)
    N = rules.N
    if cfg["coeff"]["kind"] == "grid":
        grid, plane0 = api.make_grid(rules, cfg["coeff"]["seed"], cfg["coeff"]["sigma"], 0, rules.n_rows)
        c = api.coefficient({"kind": "grid"}, grid, plane0)
        desc, host = {"kind": "grid"}, inputs.lognormal_grid(n, seed=cfg["coeff"]["seed"])
    else:
        desc, host = inputs.coefficient(cfg["coeff"], d), None
        c = api.coefficient(desc)
    u = np.random.default_rng(17).standard_normal(rules.n_rows)
    y = api.apply(rules, c, torch.from_numpy(u).cuda())
    torch.cuda.synchronize()
    rng = np.random.default_rng(9)
    edge = list(range(0, 2 * p + 2)) + list(range(N - 2 * p - 2, N))
    rows = np.array(sorted({sum(int(rng.choice(edge) if rng.random() < 0.5 else rng.integers(0, N)) * N ** a
                                for a in range(d)) for _ in range(120)}))
    A = oasm.assemble_rows(p, n, d, rows, desc, grid=host)
    absA = oasm.assemble_rows(p, n, d, rows, desc, grid=host, absolute=True)
    for kind in ("mass", "stiffness"):
        ref, scale = [], []
        for i, r in enumerate(rows):
            cols = oasm.ell_columns(p, n, d, int(r))
            ok = cols >= 0
            ref.append(A[kind][i][ok] @ u[cols[ok]])
            scale.append(absA[kind][i][ok] @ np.abs(u[cols[ok]]))
        check(y[kind].cpu().numpy()[rows], np.array(ref), np.array(scale), (name, kind))


def test_load_and_apply_ragged_ranges_bitwise():
    """Row ranges that start / end inside a z-plane and straddle the load kernel's 32-plane
    chunks and 16-row tiles (N = 39) give exactly the full-range rows (per-row arithmetic does
    not depend on the launch), for the load vector and the matrix-free product."""
    from paper_1710_01048_b200 import api, wgq
    p, n, d = 3, 36, 3
    rules = wgq.Rules(p, n, d)
    N = rules.N
    grid = torch.from_numpy(np.ascontiguousarray(inputs.lognormal_grid(n, seed=21, dim=d))).cuda()
    c = api.coefficient({"kind": "grid"}, grid, 0)
    u = torch.randn(rules.n_rows, dtype=torch.float64, device="cuda")
    b_full = api.assemble_load(rules, c)
    y_full = api.apply(rules, c, u)
    cuts = [0, 5 * N * N + 17, 7 * N * N + 4 * N + 30, 12 * N * N + 25, 31 * N * N + 3 * N + 1, 33 * N * N,
            33 * N * N + N + 38, rules.n_rows]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        b = api.assemble_load(rules, c, lo, hi)
        y = api.apply(rules, c, u, ("mass", "stiffness"), lo, hi)
        torch.cuda.synchronize()
        assert torch.equal(b, b_full[lo:hi]), (lo, hi)
        for k in ("mass", "stiffness"):
            assert torch.equal(y[k], y_full[k][lo:hi]), (lo, hi, k)
    rows = np.array([0, 5 * N * N + 17, 31 * N * N + 3 * N, 33 * N * N - 1, rules.n_rows - 1])
    ref = oops.load_rows(p, n, d, rows, {"kind": "grid", "seed": 21, "sigma": 0.5},
                         grid=inputs.lognormal_grid(n, seed=21, dim=d))
    got = b_full.cpu().numpy()[rows]
    check(got, ref, np.abs(ref), "load ragged sample")


def test_load_full_size_c3_sampled_rows():
    """C3's mesh and Fourier-lognormal coefficient (the 2D tensor-core kernel in load mode plus the
    generic shell pass): every boundary row class plus random rows against the oracle."""
    from paper_1710_01048_b200 import api, wgq
    cfg = inputs.config("C3")
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    rules = wgq.Rules(p, n, d)
    desc = inputs.coefficient(cfg["coeff"], d)
    b = api.assemble_load(rules, api.coefficient(desc))
    torch.cuda.synchronize()
    N = rules.N
    rng = np.random.default_rng(6)
    edge = list(range(0, 2 * p + 2)) + list(range(N - 2 * p - 2, N))
    rows = np.array(sorted({sum(int(rng.choice(edge) if rng.random() < 0.5 else rng.integers(0, N)) * N ** a
                                for a in range(d)) for _ in range(400)}))
    ref = oops.load_rows(p, n, d, rows, desc)
    check(b.cpu().numpy()[rows], ref, np.abs(ref), "C3 load")


@pytest.mark.parametrize("p", [2, 3])
def test_load_grid_chunks_slabs_and_alignment(p):
    """3D GRID load vector on a mesh that spans several x chunks and z chunks of the pencil kernel
    (n = 100): whole x-lines at the mesh faces, at the chunk seams and inside against the oracle;
    the same vector from an 8-byte-misaligned copy of the grid (the bulk loader's odd-parity rows)
    and, bitwise, from grid slabs (plane0 != 0, misaligned when plane0 is odd) for row ranges
    that start and end inside z-planes."""
    from paper_1710_01048_b200 import api, wgq
    n, d = 100, 3
    rules = wgq.Rules(p, n, d)
    N = rules.N
    host = np.ascontiguousarray(inputs.lognormal_grid(n, seed=33, dim=d))
    grid = torch.from_numpy(host).cuda()
    b = api.assemble_load(rules, api.coefficient({"kind": "grid"}, grid, 0))
    shifted = torch.empty(grid.numel() + 1, dtype=torch.float64, device="cuda")
    shifted[1:] = grid.reshape(-1)
    gmis = shifted[1:].view(grid.shape)
    assert gmis.data_ptr() % 16 != grid.data_ptr() % 16
    b2 = api.assemble_load(rules, api.coefficient({"kind": "grid"}, gmis, 0))
    torch.cuda.synchronize()
    assert torch.equal(b, b2)
    seam = sorted({0, 1, 2, p, p + 1, 2 * p, 34, 35, 36, 69, 70, 71, 89, 90, 91, 92, 93, N - 3, N - 2, N - 1})
    rows = np.array([(i3 * N + i2) * N + i1 for i3 in seam[::2] for i2 in seam[1::2] for i1 in range(N)])
    ref = oops.load_rows(p, n, d, rows, {"kind": "grid", "seed": 33, "sigma": 0.5}, grid=host)
    check(b.cpu().numpy()[rows], ref, np.abs(ref), ("load chunks", p))
    for lo, hi in [(3 * N * N + 17, 40 * N * N + 5 * N + 2), (N * N - 1, 2 * N * N + 1),
                   (70 * N * N + N, rules.n_rows)]:
        z0, z1 = api.grid_planes_for(rules, lo, hi)
        c = api.coefficient({"kind": "grid"}, grid[z0:z1 + 1], z0)
        bs = api.assemble_load(rules, c, lo, hi)
        torch.cuda.synchronize()
        assert torch.equal(bs, b[lo:hi]), (lo, hi, z0)
