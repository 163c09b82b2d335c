"""A rules handle is shared by threads (one per stream): the per-device caches (row tables,
separable vectors, 2D shell lists) are built under the handle's mutex on first use.  Several
threads hitting a FRESH handle at once, each on its own CUDA stream, must get exactly the rows
a single caller gets."""
import threading

import numpy as np
import pytest

import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p,n,d,kind", [(3, 9, 3, "grid"), (2, 12, 2, "fourier"), (3, 20, 2, "fourier"), (3, 8, 3, "trig")])
def test_threads_share_a_fresh_handle(p, n, d, kind):
    from paper_1710_01048_b200 import api, wgq
    desc = {"grid": {"kind": "grid"},
            "fourier": inputs.coefficient({"kind": "fourier_logn", "seed": 4, "n_modes": 8, "amp": 0.3}, d),
            "trig": {"kind": "trig_sep", "c0": 1.0, "amp": 0.4, "trig": ("sin", "cos", "sin")[:d], "wavenum": (1, 2, 1)[:d]}}[kind]
    grid = torch.from_numpy(np.ascontiguousarray(inputs.lognormal_grid(n, seed=8, dim=d))).cuda() if kind == "grid" else None
    ref_rules = wgq.Rules(p, n, d)
    c = api.coefficient(desc, grid, 0)
    ref = api.assemble(ref_rules, c)
    u = torch.randn(ref_rules.n_rows, dtype=torch.float64, device="cuda")
    ref_y = api.apply(ref_rules, c, u)
    torch.cuda.synchronize()
    rules = wgq.Rules(p, n, d)                     # fresh: no device caches yet
    T = 4
    cuts = np.linspace(0, rules.n_rows, T + 1).astype(int)
    results, errors = [None] * T, []

    def work(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                lo, hi = int(cuts[t]), int(cuts[t + 1])
                out = api.assemble(rules, c, ("mass", "stiffness"), lo, hi, stream=s)
                y = api.apply(rules, c, u, ("mass", "stiffness"), lo, hi, stream=s)
                b = api.assemble_load(rules, c, lo, hi, stream=s)
            s.synchronize()
            results[t] = (lo, hi, out, y, b)
        except Exception as e:                   # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(t,)) for t in range(T)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    ref_b = api.assemble_load(ref_rules, c)
    torch.cuda.synchronize()
    for lo, hi, out, y, b in results:
        for k in ("mass", "stiffness"):
            assert torch.equal(out[k], ref[k][lo:hi]), (lo, hi, k)
            assert torch.equal(y[k], ref_y[k][lo:hi]), (lo, hi, k)
        assert torch.equal(b, ref_b[lo:hi])
