"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck).

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1710_01048_b200 import api, wgq  # noqa: E402


def run(p, n, d, desc, kinds=("mass", "stiffness")):
    r = wgq.Rules(p, n, d)
    gt = None
    if desc["kind"] == "grid":
        gt = torch.from_numpy(np.ascontiguousarray(inputs.lognormal_grid(n, seed=3, dim=d))).cuda()
    c = api.coefficient(desc, gt, 0)
    api.assemble(r, c, kinds)
    N = r.N
    lo, hi = min(5, r.n_rows // 3), r.n_rows - min(4, r.n_rows // 3)
    api.assemble_csr(r, c, kinds, lo, hi)
    api.assemble(r, c, kinds, lo, hi, ld=r.stencil + 1)
    api.assemble_load(r, c)
    u = torch.randn(r.n_rows, dtype=torch.float64, device="cuda")
    api.apply(r, c, u, kinds)
    if d >= 2:                                           # a slab with u holding only its halo
        pr = N ** (d - 1)
        z0, z1 = 1, min(N, 3)
        ulo, uhi = max(0, z0 - p) * pr, min(N, z1 + p) * pr
        api.apply(r, c, u[ulo:uhi], kinds, z0 * pr, z1 * pr, u_row0=ulo)
    torch.cuda.synchronize()


four = lambda d: inputs.coefficient({"kind": "fourier_logn", "seed": 1, "n_modes": 8, "amp": 0.3}, d)
trig = lambda d: {"kind": "trig_sep", "c0": 1.0, "amp": 0.4, "trig": ("sin", "cos", "sin")[:d], "wavenum": (1, 2, 1)[:d]}
for p in (2, 3):
    run(p, 7, 3, {"kind": "grid"})                       # line kernels (ELL, CSR, padded ld), apply, load
    run(p, 4, 3, {"kind": "grid"})
    run(p, 9, 2, four(2))                                # 2D tensor-core kernel + shell
    run(p, 6, 3, trig(3))                                # separable 3D
    run(p, 8, 2, trig(2))                                # separable 2D
    run(p, 5, 3, four(3))                                # generic
    run(p, 11, 1, {"kind": "const", "c0": 1.0})
run(3, 21, 2, four(2))                                   # fused 2D FOURIER launch: interior, frame, shell items
run(3, 40, 3, {"kind": "grid"})                          # several load-tile blocks in x, y and z
for p in (2, 3):                                         # per-direction element counts
    r = wgq.Rules(p, (7, 9, 11), 3)
    gt = api.make_grid(r, 5, 0.5, 0, r.n_rows)[0]
    c = api.coefficient({"kind": "grid"}, gt, 0)
    api.assemble(r, c, ("mass", "stiffness"))
    api.assemble_load(r, c)
    api.apply(r, c, torch.randn(r.n_rows, dtype=torch.float64, device="cuda"), ("mass", "stiffness"))
    torch.cuda.synchronize()
print("sanitize case done")
