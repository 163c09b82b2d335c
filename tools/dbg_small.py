import sys; sys.path.insert(0, '.')
import numpy as np, torch
from oracle import assemble as oasm
from paper_1710_01048_b200 import api, wgq
np.set_printoptions(precision=6, linewidth=200, suppress=True)
for (p, d, n) in [(2, 1, 2), (2, 1, 3), (2, 2, 2), (3, 1, 3)]:
    r = wgq.Rules(p, n, d)
    for cls in range(p + 1):
        print(p, n, "cls", cls, "K", wgq.wgq_rules_query(r, cls, 1)[:2])
    out = api.assemble(r, api.coefficient({"kind": "const", "c0": 1.0}))
    torch.cuda.synchronize()
    ref = oasm.assemble_rows(p, n, d, np.arange(r.n_rows), {"kind": "const", "c0": 1.0})
    for k in ("mass", "stiffness"):
        g = out[k].cpu().numpy()
        err = np.abs(g - ref[k]).max(axis=1)
        print(p, d, n, k, "row errs", err)
        if err.max() > 1e-12 and d == 1:
            print("gpu\n", g, "\nref\n", ref[k])
