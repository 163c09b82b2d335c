"""Out-of-bounds write guards (compute-sanitizer is not available on this pool): every kernel
family writes its outputs into views of larger buffers whose guard regions hold a sentinel;
after assembly (ELL, padded ELL, CSR), load vector and matrix-free product the sentinels
must be intact and every in-range element must have been written."""
import numpy as np
import pytest

import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SENT = -7.25e300
G = 4096                                     # guard elements on each side


def guarded(n_elems):
    buf = torch.full((n_elems + 2 * G,), SENT, dtype=torch.float64, device="cuda")
    return buf, buf[G:G + n_elems]


def check_guards(buf, n_elems, what):
    b = buf.cpu().numpy()
    assert np.all(b[:G] == SENT) and np.all(b[G + n_elems:] == SENT), what
    assert not np.any(b[G:G + n_elems] == SENT), what + ": unwritten elements"


def cases():
    four = lambda d: inputs.coefficient({"kind": "fourier_logn", "seed": 1, "n_modes": 8, "amp": 0.3}, d)
    trig = lambda d: {"kind": "trig_sep", "c0": 1.0, "amp": 0.4, "trig": ("sin", "cos", "sin")[:d], "wavenum": (1, 2, 1)[:d]}
    out = []
    for p in (2, 3):
        out += [(p, 7, 3, {"kind": "grid"}), (p, 4, 3, {"kind": "grid"}), (p, 9, 2, four(2)), (p, 6, 3, trig(3)),
                (p, 8, 2, trig(2)), (p, 5, 3, four(3)), (p, 11, 1, {"kind": "const", "c0": 1.0})]
    # lines of several tiles (assembly: 12 rows, apply: 24, load: 16 x 16 tiles, 32-plane chunks)
    out += [(3, 30, 3, {"kind": "grid"}), (2, 35, 3, {"kind": "grid"})]
    return out


@pytest.mark.parametrize("case", range(16))
def test_no_out_of_bounds_writes(case):
    from paper_1710_01048_b200 import api, wgq
    p, n, d, desc = cases()[case]
    r = wgq.Rules(p, n, d)
    gt = None
    if desc["kind"] == "grid":
        gt = torch.from_numpy(np.ascontiguousarray(inputs.lognormal_grid(n, seed=3, dim=d))).cuda()
    c = api.coefficient(desc, gt, 0)
    lo, hi = min(5, r.n_rows // 3), r.n_rows - min(4, r.n_rows // 3)
    rows = hi - lo
    for ld in (r.stencil, r.stencil + 1):
        bm, vm = guarded(rows * ld)
        bk, vk = guarded(rows * ld)
        out = {"mass": vm.view(rows, ld), "stiffness": vk.view(rows, ld)}
        api.assemble(r, c, ("mass", "stiffness"), lo, hi, out=out)
        torch.cuda.synchronize()
        if ld == r.stencil:
            check_guards(bm, rows * ld, f"ELL mass {p, n, d}")
            check_guards(bk, rows * ld, f"ELL stiffness {p, n, d}")
        else:                                   # padded ld: slot ld-1 of every row is not written
            for b in (bm, bk):
                arr = b.cpu().numpy()
                assert np.all(arr[:G] == SENT) and np.all(arr[G + rows * ld:] == SENT)
                body = arr[G:G + rows * ld].reshape(rows, ld)
                assert not np.any(body[:, :-1] == SENT) and np.all(body[:, -1] == SENT)
    nnz = wgq.wgq_nnz(r, lo, hi)
    row_ptr = torch.empty(rows + 1, dtype=torch.int64, device="cuda")
    col_idx = torch.empty(nnz, dtype=torch.int32, device="cuda")
    wgq.wgq_csr_structure(r, lo, hi, row_ptr, col_idx)
    bm, vm = guarded(nnz)
    bk, vk = guarded(nnz)
    wgq.wgq_assemble_mass_stiffness(r, c, wgq.make_out(vm, lo, hi, ld=0, layout=wgq.WGQ_CSR, row_ptr=row_ptr),
                                    wgq.make_out(vk, lo, hi, ld=0, layout=wgq.WGQ_CSR, row_ptr=row_ptr))
    torch.cuda.synchronize()
    check_guards(bm, nnz, f"CSR mass {p, n, d}")
    check_guards(bk, nnz, f"CSR stiffness {p, n, d}")
    bb, vb = guarded(rows)
    api.assemble_load(r, c, lo, hi, out=vb)
    torch.cuda.synchronize()
    check_guards(bb, rows, f"load {p, n, d}")
    u = torch.randn(r.n_rows, dtype=torch.float64, device="cuda")
    bym, ym = guarded(rows)
    byk, yk = guarded(rows)
    wgq.wgq_apply(r, c, u, 0, lo, hi, ym, yk)
    torch.cuda.synchronize()
    check_guards(bym, rows, f"apply M {p, n, d}")
    check_guards(byk, rows, f"apply K {p, n, d}")


@pytest.mark.parametrize("p,n,d,kind", [(3, 6, 3, "grid"), (2, 9, 2, "fourier"), (3, 5, 3, "trig"), (2, 7, 1, "const")])
def test_empty_row_ranges_write_nothing(p, n, d, kind):
    """row_begin == row_end (a rank with no rows) is a no-op for every entry point, at any row."""
    from paper_1710_01048_b200 import api, wgq
    r = wgq.Rules(p, n, d)
    gt = None
    if kind == "grid":
        gt = torch.from_numpy(np.ascontiguousarray(inputs.lognormal_grid(n, seed=3, dim=d))).cuda()
    desc = {"grid": {"kind": "grid"}, "const": {"kind": "const", "c0": 1.0},
            "trig": {"kind": "trig_sep", "c0": 1.0, "amp": 0.4, "trig": ("sin", "cos", "sin")[:d], "wavenum": (1, 2, 1)[:d]},
            "fourier": inputs.coefficient({"kind": "fourier_logn", "seed": 1, "n_modes": 8, "amp": 0.3}, d)}[kind]
    c = api.coefficient(desc, gt, 0)
    for at in (0, r.n_rows // 2, r.n_rows):
        buf, view = guarded(0)
        out = {"mass": view.view(0, r.stencil), "stiffness": view.view(0, r.stencil)}
        api.assemble(r, c, ("mass", "stiffness"), at, at, out=out)
        row_ptr = torch.full((1,), 123, dtype=torch.int64, device="cuda")
        wgq.wgq_csr_structure(r, at, at, row_ptr, None)           # row_ptr = [0]: slab-local, from 0
        api.assemble_load(r, c, at, at, out=view)
        u = torch.randn(r.n_rows, dtype=torch.float64, device="cuda")
        y = api.apply(r, c, u, ("mass", "stiffness"), at, at)
        torch.cuda.synchronize()
        assert all(v.numel() == 0 for v in y.values())
        assert int(row_ptr[0].item()) == 0
        check_guards(buf, 0, f"empty range at {at}")
