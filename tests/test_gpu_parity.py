"""GPU parity: the CUDA path (through the C-ABI) against the oracle, element by element.

Tolerance (north_star, R12): relative Frobenius <= 1e-12 and max entrywise
relative <= 1e-10, the entrywise denominator being max(|o|, 1e-14 max_row|o|, F) with
F = 64 eps / 1e-10 * sum_k |term_k| (the oracle's absolute-value assembly): an entry that is
smaller than the rounding scale of its own terms (cancellation, mathematically-zero entries)
is held to that rounding scale instead of to a relative error it cannot have in FP64.
"""
import numpy as np
import pytest

import inputs
from oracle import assemble as oasm

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from parity import REL_E, REL_F, compare  # noqa: E402,F401


def coeff_cases(d, n):
    out = [("const", {"kind": "const", "c0": 1.0}),
           ("trig", {"kind": "trig_sep", "c0": 1.0, "amp": 0.5, "trig": ("sin", "cos", "sin")[:d], "wavenum": (1, 1, 2)[:d]}),
           ("fourier", inputs.coefficient({"kind": "fourier_logn", "seed": inputs.SEED, "n_modes": 8, "amp": 0.3}, d)),
           ("grid", {"kind": "grid", "seed": 3, "sigma": 0.5})]
    return out


def gpu_assemble(p, n, d, desc, kinds=("mass", "stiffness"), row_begin=0, row_end=None, bnd=0, host_grid=None,
                 plane0=0, ld=None):
    from paper_1710_01048_b200 import api, wgq
    rules = wgq.Rules(p, n, d, bnd)
    grid_t = None
    if desc["kind"] == "grid":
        grid_t = torch.from_numpy(np.ascontiguousarray(host_grid)).cuda()
    c = api.coefficient(desc, grid_t, plane0)
    out = api.assemble(rules, c, kinds, row_begin, row_end, ld=ld)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}, rules


SMALL = [(2, 1, 64), (3, 1, 33), (2, 2, 13), (3, 2, 11), (2, 3, 7), (3, 3, 6), (3, 3, 3), (2, 2, 2)]


@pytest.mark.parametrize("p,d,n", SMALL)
def test_all_rows_all_coefficients(p, d, n):
    N = n + p
    rows = np.arange(N ** d)
    for name, desc in coeff_cases(d, n):
        grid = inputs.lognormal_grid(n, seed=desc.get("seed", 1), dim=d) if name == "grid" else None
        g, _ = gpu_assemble(p, n, d, desc, host_grid=grid)
        ref = oasm.assemble_rows(p, n, d, rows, desc, grid=grid)
        sc = oasm.assemble_rows(p, n, d, rows, desc, grid=grid, absolute=True)
        for k in ("mass", "stiffness"):
            compare(g[k], ref[k], (p, d, n, name, k), sc[k])


@pytest.mark.parametrize("p,d,n,kind", [(2, 2, 9, "trig"), (3, 3, 4, "trig"), (3, 2, 10, "fourier"), (2, 2, 7, "fourier")])
def test_gl_boundary_mode(p, d, n, kind):
    """WGQ_BND_GL: every boundary class uses GL per element (up to p(p+1) nodes), which sends
    the 2D FOURIER rows touching them through the generic shell pass."""
    N = n + p
    rows = np.arange(N ** d)
    if kind == "trig":
        desc = {"kind": "trig_sep", "c0": 1.0, "amp": 0.5, "trig": ("sin",) * d, "wavenum": (1,) * d}
    else:
        desc = inputs.coefficient({"kind": "fourier_logn", "seed": 11, "n_modes": 8, "amp": 0.3}, d)
    g, _ = gpu_assemble(p, n, d, desc, bnd=1)
    ref = oasm.assemble_rows(p, n, d, rows, desc, mode="gl")
    sc = oasm.assemble_rows(p, n, d, rows, desc, mode="gl", absolute=True)
    for k in ("mass", "stiffness"):
        compare(g[k], ref[k], ("gl", k), sc[k])


def test_constant_coefficient_exact_1d_c1():
    """C1: 1D p=2 n=64 c=1 mass against the exact Galerkin matrix (closed form via scipy)."""
    from wgq_exact import exact_1d, to_ell
    g, _ = gpu_assemble(2, 64, 1, {"kind": "const", "c0": 1.0}, kinds=("mass",))
    M, _ = exact_1d(2, 64)
    compare(g["mass"], to_ell(M, 2, 64, 1), "C1")


def test_slabs_bitwise_equal_and_padded_ld():
    p, d, n = 3, 3, 7
    N = n + p
    desc = {"kind": "grid", "seed": 9, "sigma": 0.5}
    grid = inputs.lognormal_grid(n, seed=9)
    full, _ = gpu_assemble(p, n, d, desc, host_grid=grid)
    b = [0, 7 * N * N, 8 * N * N + 5, N ** 3]            # uneven, ragged slab boundaries
    for lo, hi in zip(b[:-1], b[1:]):
        z0, z1 = lo // (N * N), (hi - 1) // (N * N)
        pl, ph = max(0, z0 - p), min(n, z1 + 1)
        part, _ = gpu_assemble(p, n, d, desc, row_begin=lo, row_end=hi, host_grid=grid[pl:ph + 1], plane0=pl, ld=344)
        for k in ("mass", "stiffness"):
            assert np.array_equal(part[k][:, :343], full[k][lo:hi]), (lo, hi, k)


@pytest.mark.parametrize("p,d,n,kind", [(2, 3, 5, "trig"), (3, 2, 9, "fourier"), (2, 2, 6, "fourier"),
                                        (3, 1, 12, "const"), (3, 3, 4, "fourier"), (3, 3, 9, "grid"),
                                        (2, 3, 7, "grid"), (3, 3, 4, "grid")])
def test_csr_matches_ell(p, d, n, kind):
    """CSR values equal the ELL values at the structural columns, for every kernel family
    (separable, 2D tensor-core FOURIER incl. its shell pass, generic)."""
    from paper_1710_01048_b200 import api, wgq
    rules = wgq.Rules(p, n, d)
    if kind == "trig":
        desc = {"kind": "trig_sep", "c0": 1.0, "amp": 0.3, "trig": ("sin",) * d, "wavenum": (1,) * d}
    elif kind == "const":
        desc = {"kind": "const", "c0": 2.5}
    elif kind == "grid":
        desc = {"kind": "grid", "seed": 21, "sigma": 0.5}
    else:
        desc = inputs.coefficient({"kind": "fourier_logn", "seed": 7, "n_modes": 8, "amp": 0.3}, d)
    gt = None
    if kind == "grid":
        gt = torch.from_numpy(np.ascontiguousarray(inputs.lognormal_grid(n, seed=21, dim=d))).cuda()
    c = api.coefficient(desc, gt, 0)
    ell = api.assemble(rules, c)
    lo, hi = min(17, rules.n_rows // 4), rules.n_rows - min(11, rules.n_rows // 4)
    row_ptr, col_idx, vals = api.assemble_csr(rules, c, row_begin=lo, row_end=hi)
    torch.cuda.synchronize()
    rp, ci = row_ptr.cpu().numpy(), col_idx.cpu().numpy()
    for k in ("mass", "stiffness"):
        e = ell[k].cpu().numpy()
        v = vals[k].cpu().numpy()
        for r in range(lo, hi):
            cols = oasm.ell_columns(p, n, d, r)
            ok = cols >= 0
            seg = slice(rp[r - lo], rp[r - lo + 1])
            assert np.array_equal(ci[seg], cols[ok])
            assert np.array_equal(v[seg], e[r][ok])
    assert rp[-1] == wgq.wgq_nnz(rules, lo, hi)


@pytest.mark.parametrize("dim,n,plane0,planes", [(3, 16, 0, 17), (3, 20, 5, 9), (2, 40, 3, 20), (1, 30, 0, 31)])
def test_device_grid_generator_matches_inputs(dim, n, plane0, planes):
    from paper_1710_01048_b200 import wgq
    shape = {1: (n + 1,), 2: (planes, n + 1), 3: (planes, n + 1, n + 1)}[dim]
    g = torch.empty(shape, dtype=torch.float64, device="cuda")
    wgq.wgq_generate_grid(n, dim, inputs.SEED, 0.5, plane0, planes, g)
    torch.cuda.synchronize()
    ref = inputs.lognormal_grid(n, seed=inputs.SEED, dim=dim, plane0=plane0, planes=planes if dim > 1 else None)
    assert np.max(np.abs(g.cpu().numpy() - ref) / ref) < 1e-14


def test_row_moments_identities():
    """P9 on the GPU output: (K 1)_i = 0 and (M 1)_i = sum_k W^M_ik for all rows."""
    from paper_1710_01048_b200 import api, wgq
    p, d, n = 3, 3, 6
    N = n + p
    desc = inputs.coefficient({"kind": "fourier_logn", "seed": 5, "n_modes": 8, "amp": 0.3}, 3)
    rules = wgq.Rules(p, n, d)
    out = api.assemble(rules, api.coefficient(desc))
    mom = {}
    for k in ("mass", "stiffness"):
        m = torch.empty((N ** d, 1 + d), dtype=torch.float64, device="cuda")
        wgq.wgq_row_moments(rules, wgq.make_out(out[k], 0, N ** d), m)
        mom[k] = m.cpu().numpy()
    rows = np.arange(N ** d)
    m1, mx, kx = oasm.row_weight_sums(p, n, d, rows, desc)
    scaleM = np.abs(out["mass"].cpu().numpy()).max(axis=1)
    scaleK = np.abs(out["stiffness"].cpu().numpy()).max(axis=1)
    assert np.max(np.abs(mom["mass"][:, 0] - m1) / scaleM) < 1e-13
    assert np.max(np.abs(mom["stiffness"][:, 0]) / scaleK) < 1e-13
    for a in range(d):
        assert np.max(np.abs(mom["mass"][:, 1 + a] - mx[:, a]) / scaleM) < 1e-13
        assert np.max(np.abs(mom["stiffness"][:, 1 + a] - kx[:, a]) / scaleK) < 1e-13


@pytest.mark.parametrize("n", [9, 10, 21, 40])
def test_fourier2d_interior_kernel(n):
    """C3's kernel pair (p = 3, 2D FOURIER): the class-I interior kernel (2 lines x row pairs,
    chunks of 8 pairs) plus the frame kernel, over whole meshes whose interior has an odd / even
    number of lines and rows and several chunks, and over ragged row ranges that start and end
    inside lines (slabs), ELL with padded ld and CSR."""
    from paper_1710_01048_b200 import api, wgq
    p, d = 3, 2
    N = n + p
    desc = inputs.coefficient({"kind": "fourier_logn", "seed": 13, "n_modes": 8, "amp": 0.3}, d)
    rows = np.arange(N ** d)
    ref = oasm.assemble_rows(p, n, d, rows, desc)
    sc = oasm.assemble_rows(p, n, d, rows, desc, absolute=True)
    g, _ = gpu_assemble(p, n, d, desc)
    for k in ("mass", "stiffness"):
        compare(g[k], ref[k], ("f2d-int", n, k), sc[k])
    rules = wgq.Rules(p, n, d)
    c = api.coefficient(desc)
    for lo, hi in ((7 * N + 3, 9 * N + 8), (N + 5, N * N - N - 2), (6 * N + 6, 6 * N + 9)):
        out = api.assemble(rules, c, row_begin=lo, row_end=hi, ld=50)
        rp, ci, vals = api.assemble_csr(rules, c, row_begin=lo, row_end=hi)
        torch.cuda.synchronize()
        rpn = rp.cpu().numpy()
        for k in ("mass", "stiffness"):
            e = out[k].cpu().numpy()
            assert np.array_equal(e[:, :49], g[k][lo:hi]), (lo, hi, k)
            v = vals[k].cpu().numpy()
            for r in range(lo, hi):
                cols = oasm.ell_columns(p, n, d, r)
                assert np.array_equal(v[rpn[r - lo]:rpn[r - lo + 1]], g[k][r][cols >= 0]), (r, k)


@pytest.mark.parametrize("p,n", [(2, 7), (3, 6)])
def test_gl_boundary_mode_grid_3d(p, n):
    """WGQ_BND_GL ("or one can use standard Gauss rules there") with the GRID
    coefficient in 3D: the line kernel (ELL, compact and padded ld), its CSR runs, the load
    vector and the matrix-free product against the oracle in mode "gl"."""
    from paper_1710_01048_b200 import api, wgq
    d = 3
    N = n + p
    rows = np.arange(N ** d)
    desc = {"kind": "grid", "seed": 23, "sigma": 0.5}
    grid = inputs.lognormal_grid(n, seed=23)
    ref = oasm.assemble_rows(p, n, d, rows, desc, grid=grid, mode="gl")
    sc = oasm.assemble_rows(p, n, d, rows, desc, grid=grid, mode="gl", absolute=True)
    s3 = (2 * p + 1) ** 3
    for ld in (None, s3 + 3):
        g, _ = gpu_assemble(p, n, d, desc, bnd=wgq.WGQ_BND_GL, host_grid=grid, ld=ld)
        for k in ("mass", "stiffness"):
            compare(g[k][:, :s3], ref[k], ("gl-grid", p, n, ld, k), sc[k])
    rules = wgq.Rules(p, n, d, wgq.WGQ_BND_GL)
    c = api.coefficient(desc, torch.from_numpy(grid).cuda(), 0)
    rp, ci, vals = api.assemble_csr(rules, c)
    b = api.assemble_load(rules, c)
    u = np.random.default_rng(3).standard_normal(N ** d)
    y = api.apply(rules, c, torch.from_numpy(u).cuda())
    torch.cuda.synchronize()
    rpn = rp.cpu().numpy()
    for k in ("mass", "stiffness"):
        v = vals[k].cpu().numpy()
        for r in rows:
            cols = oasm.ell_columns(p, n, d, r)
            assert np.array_equal(v[rpn[r]:rpn[r + 1]], g[k][r][:s3][cols >= 0]), (r, k)
    from oracle import operators as oops
    bref = oops.load_rows(p, n, d, rows, desc, grid=grid, mode="gl")
    compare(b.cpu().numpy(), bref, ("gl-grid load", p, n), rowwise=False)
    for k in ("mass", "stiffness"):
        yref = oops.apply_rows(p, n, d, rows, desc, u, k, grid=grid, mode="gl")
        scale = np.array([np.abs(sc[k][i][oasm.ell_columns(p, n, d, r) >= 0]) @
                          np.abs(u[oasm.ell_columns(p, n, d, r)[oasm.ell_columns(p, n, d, r) >= 0]])
                          for i, r in enumerate(rows)])
        compare(y[k].cpu().numpy(), yref, ("gl-grid apply", p, n, k), scale, rowwise=False)


@pytest.mark.parametrize("p,n,bnd", [(3, 10, 0), (2, 9, 1), (3, 12, 1)])
def test_fourier2d_shell_rows_ragged_ranges(p, n, bnd):
    """The 2D FOURIER shell pass (rows touching a GL-fallback class, generated on the device per
    call) over row ranges that start and end inside lines, for the assembly, the load vector and
    the matrix-free product: every range reproduces the whole-mesh rows bitwise."""
    from paper_1710_01048_b200 import api, wgq
    d = 2
    N = n + p
    rules = wgq.Rules(p, n, d, bnd)
    c = api.coefficient(inputs.coefficient({"kind": "fourier_logn", "seed": 29, "n_modes": 8, "amp": 0.3}, d))
    full = api.assemble(rules, c)
    bfull = api.assemble_load(rules, c)
    u = torch.from_numpy(np.random.default_rng(2).standard_normal(N * N)).cuda()
    yfull = api.apply(rules, c, u)
    for lo, hi in ((1, N + 2), (N - 1, 2 * N + 1), (3 * N + 1, N * N - 1), (N * N - N - 1, N * N)):
        part = api.assemble(rules, c, row_begin=lo, row_end=hi)
        b = api.assemble_load(rules, c, lo, hi)
        y = api.apply(rules, c, u, row_begin=lo, row_end=hi)
        torch.cuda.synchronize()
        for k in ("mass", "stiffness"):
            assert torch.equal(part[k], full[k][lo:hi]), (lo, hi, k)
            assert torch.equal(y[k], yfull[k][lo:hi]), (lo, hi, k)
        assert torch.equal(b, bfull[lo:hi]), (lo, hi)
