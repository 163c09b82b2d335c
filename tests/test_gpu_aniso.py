"""GPU parity on meshes with a different element count per direction (eq:Gmap3 P:113-120:
each parameter direction has its own knot vector with n_EL^i elements; eq:DimMulti P:134-136),
through the C-ABI (wgq_build_rules_ex2): assembly (ELL and CSR), load vector, matrix-free
product, row moments and the device grid generator, for every coefficient kind, against the
oracle (tests/parity.py tolerances)."""
import numpy as np
import pytest

import inputs
from oracle import assemble as oasm
from oracle import operators as oops

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from parity import compare  # noqa: E402

MESHES = [(2, (7, 9, 11), 3), (3, (5, 4, 6), 3), (3, (5, 13), 2), (2, (12, 5), 2), (3, (9,), 1)]


def coeff_cases(d):
    return [("const", {"kind": "const", "c0": 1.3}),
            ("trig", {"kind": "trig_sep", "c0": 1.0, "amp": 0.5, "trig": ("sin", "cos", "sin")[:d],
                      "wavenum": (1, 2, 1)[:d]}),
            ("fourier", inputs.coefficient({"kind": "fourier_logn", "seed": 31, "n_modes": 8, "amp": 0.3}, d)),
            ("grid", {"kind": "grid", "seed": 8, "sigma": 0.5})]


def _coef(desc, n, d):
    from paper_1710_01048_b200 import api
    grid = inputs.lognormal_grid(n, seed=desc["seed"], dim=d) if desc["kind"] == "grid" else None
    gt = torch.from_numpy(np.ascontiguousarray(grid)).cuda() if grid is not None else None
    return api.coefficient(desc, gt, 0), grid


@pytest.mark.parametrize("p,n,d", MESHES)
def test_aniso_assembly_all_coefficients(p, n, d):
    from paper_1710_01048_b200 import api, wgq
    rules = wgq.Rules(p, n, d)
    assert rules.Ns == tuple(v + p for v in n) and rules.n_rows == int(np.prod(rules.Ns))
    rows = np.arange(rules.n_rows)
    for name, desc in coeff_cases(d):
        c, grid = _coef(desc, n, d)
        out = api.assemble(rules, c)
        torch.cuda.synchronize()
        ref = oasm.assemble_rows(p, n, d, rows, desc, grid=grid)
        sc = oasm.assemble_rows(p, n, d, rows, desc, grid=grid, absolute=True)
        for k in ("mass", "stiffness"):
            compare(out[k].cpu().numpy(), ref[k], ("aniso", p, n, name, k), sc[k])
        # CSR: the closed-form structure per direction, values = the ELL values
        lo, hi = 3, rules.n_rows - 2
        rp, ci, vals = api.assemble_csr(rules, c, row_begin=lo, row_end=hi)
        torch.cuda.synchronize()
        rpn, cin = rp.cpu().numpy(), ci.cpu().numpy()
        assert rpn[-1] == wgq.wgq_nnz(rules, lo, hi)
        for k in ("mass", "stiffness"):
            e, v = out[k].cpu().numpy(), vals[k].cpu().numpy()
            for r in range(lo, hi):
                cols = oasm.ell_columns(p, n, d, r)
                seg = slice(rpn[r - lo], rpn[r - lo + 1])
                assert np.array_equal(cin[seg], cols[cols >= 0]), (name, r)
                assert np.array_equal(v[seg], e[r][cols >= 0]), (name, r, k)


@pytest.mark.parametrize("p,n,d", MESHES[:4])
def test_aniso_load_apply_and_moments(p, n, d):
    from paper_1710_01048_b200 import api, wgq
    rules = wgq.Rules(p, n, d)
    rows = np.arange(rules.n_rows)
    u = np.random.default_rng(1).standard_normal(rules.n_rows)
    for name, desc in coeff_cases(d):
        c, grid = _coef(desc, n, d)
        b = api.assemble_load(rules, c)
        y = api.apply(rules, c, torch.from_numpy(u).cuda())
        out = api.assemble(rules, c)
        torch.cuda.synchronize()
        compare(b.cpu().numpy(), oops.load_rows(p, n, d, rows, desc, grid=grid), ("aniso load", n, name), rowwise=False)
        sc = oasm.assemble_rows(p, n, d, rows, desc, grid=grid, absolute=True)
        cols = [oasm.ell_columns(p, n, d, r) for r in rows]
        for k in ("mass", "stiffness"):
            yref = oops.apply_rows(p, n, d, rows, desc, u, k, grid=grid)
            scale = np.array([np.abs(sc[k][i][c_ >= 0]) @ np.abs(u[c_[c_ >= 0]]) for i, c_ in enumerate(cols)])
            compare(y[k].cpu().numpy(), yref, ("aniso apply", n, name, k), scale, rowwise=False)
        # P9 row moments against the oracle's weighted sums (M 1, M g^a, K 1 = 0, K g^a)
        m1, mx, kx = oasm.row_weight_sums(p, n, d, rows, desc, grid=grid)
        for k in ("mass", "stiffness"):
            mom = torch.empty((rules.n_rows, 1 + d), dtype=torch.float64, device="cuda")
            wgq.wgq_row_moments(rules, wgq.make_out(out[k], 0, rules.n_rows), mom)
            mom = mom.cpu().numpy()
            rmax = out[k].abs().amax(dim=1).cpu().numpy()
            if k == "mass":
                assert np.max(np.abs(mom[:, 0] - m1) / rmax) < 1e-13
                for a in range(d):
                    assert np.max(np.abs(mom[:, 1 + a] - mx[:, a]) / rmax) < 1e-13
            else:
                assert np.max(np.abs(mom[:, 0]) / rmax) < 1e-12
                for a in range(d):
                    assert np.max(np.abs(mom[:, 1 + a] - kx[:, a]) / rmax) < 1e-13


@pytest.mark.parametrize("n,dim,plane0,planes", [((9, 6, 7), 3, 0, 8), ((9, 6, 7), 3, 2, 4), ((11, 5), 2, 1, 4)])
def test_aniso_device_grid_generator(n, dim, plane0, planes):
    from paper_1710_01048_b200 import wgq
    shape = (planes, n[1] + 1, n[0] + 1) if dim == 3 else (planes, n[0] + 1)
    g = torch.empty(shape, dtype=torch.float64, device="cuda")
    wgq.wgq_generate_grid(n, dim, inputs.SEED, 0.5, plane0, planes, g)
    torch.cuda.synchronize()
    ref = inputs.lognormal_grid(n, seed=inputs.SEED, dim=dim, plane0=plane0, planes=planes)
    assert np.max(np.abs(g.cpu().numpy() - ref) / ref) < 1e-14


def test_aniso_slabs_bitwise():
    """z-slabs of an anisotropic 3D GRID assembly (each with its own generated vertex slab)
    reproduce the whole-mesh rows bitwise."""
    from paper_1710_01048_b200 import api, wgq
    p, n, d = 3, (6, 8, 7), 3
    rules = wgq.Rules(p, n, d)
    g, lo = api.make_grid(rules, 5, 0.5, 0, rules.n_rows)
    full = api.assemble(rules, api.coefficient({"kind": "grid"}, g, lo))
    for r in range(3):
        b, e = api.slab_rows(rules.Ns, d, r, 3)
        gs, l0 = api.make_grid(rules, 5, 0.5, b, e)
        part = api.assemble(rules, api.coefficient({"kind": "grid"}, gs, l0), row_begin=b, row_end=e)
        torch.cuda.synchronize()
        for k in ("mass", "stiffness"):
            assert torch.equal(part[k], full[k][b:e]), (r, k)
