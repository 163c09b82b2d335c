"""wgq_assemble_host (the end-to-end path bench.py's e2e number goes through): host coefficient
in, host ELL out, chunked two-stream pipeline — must give exactly the device assembly's rows for
any chunking, row range, padded ld and matrix selection."""
import numpy as np
import pytest

import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


class _HostGrid:
    def __init__(self, arr):
        self.arr = arr
        self.shape = arr.shape

    def data_ptr(self):
        return self.arr.ctypes.data


CASES = [
    (3, 9, 3, {"kind": "grid", "seed": 5, "sigma": 0.5}),
    (2, 7, 3, {"kind": "grid", "seed": 6, "sigma": 0.5}),
    (3, 12, 2, "fourier"),
    (2, 10, 3, {"kind": "trig_sep", "c0": 1.0, "amp": 0.4, "trig": ("sin", "cos", "sin"), "wavenum": (1, 2, 1)}),
    (3, 20, 1, {"kind": "const", "c0": 1.0}),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_host_pipeline_equals_device(case):
    from paper_1710_01048_b200 import api, wgq
    p, n, d, desc = CASES[case]
    if desc == "fourier":
        desc = inputs.coefficient({"kind": "fourier_logn", "seed": 3, "n_modes": 8, "amp": 0.3}, d)
    r = wgq.Rules(p, n, d)
    N = r.N
    grid = inputs.lognormal_grid(n, seed=desc["seed"], dim=d) if desc["kind"] == "grid" else None
    dev_coef = api.coefficient(desc, torch.from_numpy(np.ascontiguousarray(grid)).cuda() if grid is not None else None, 0)
    full = api.assemble(r, dev_coef)
    torch.cuda.synchronize()
    ref = {k: v.cpu().numpy() for k, v in full.items()}
    lo, hi = (N ** (d - 1) + 3, r.n_rows - N - 1) if d > 1 else (2, r.n_rows - 1)
    for (rb, re), chunk, ld, kinds in (((0, r.n_rows), 0, r.stencil, ("mass", "stiffness")),
                                       ((lo, hi), 37, r.stencil + 3, ("mass", "stiffness")),
                                       ((lo, hi), 5, r.stencil, ("stiffness",))):
        if desc["kind"] == "grid" and d > 1:
            pl, ph = api.grid_planes_for(r, rb, re)
            hg = np.ascontiguousarray(grid[pl:ph + 1])
            coef = wgq.make_coeff({"kind": "grid"}, grid=_HostGrid(hg), plane0=pl)
        elif desc["kind"] == "grid":
            coef = wgq.make_coeff({"kind": "grid"}, grid=_HostGrid(np.ascontiguousarray(grid)), plane0=0)
        else:
            coef = api.coefficient(desc)
        rows = re - rb
        host = {k: wgq.PinnedArray((rows, ld)) for k in kinds}
        for v in host.values():
            v.array[...] = -1.0
        wgq.wgq_assemble_host(r, coef, rb, re, host["mass"].array if "mass" in host else None,
                              host["stiffness"].array if "stiffness" in host else None, ld, chunk)
        for k in kinds:
            assert np.array_equal(host[k].array[:, :r.stencil], ref[k][rb:re]), (case, rb, re, chunk, k)
            if ld > r.stencil:
                assert np.all(host[k].array[:, r.stencil:] == -1.0)     # padding slots untouched
            host[k].close()
