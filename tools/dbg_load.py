import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import inputs
from oracle import operators
from paper_1710_01048_b200 import api, wgq
for (p,d,n) in [(3,2,8),(3,3,4),(2,2,9)]:
    rules = wgq.Rules(p, n, d)
    N = rules.N
    grid = inputs.lognormal_grid(n, seed=4, dim=d)
    c = api.coefficient({"kind": "grid"}, torch.from_numpy(np.ascontiguousarray(grid)).cuda(), 0)
    b = api.assemble_load(rules, c).cpu().numpy()
    ref = operators.load_rows(p, n, d, np.arange(rules.n_rows), {"kind": "grid"}, grid=grid)
    bad = np.where(np.abs(b - ref) > 1e-12 * np.abs(ref))[0]
    print(p, d, n, "bad rows", len(bad), [tuple(int(x) for x in np.unravel_index(r, (N,) * d)[::-1]) for r in bad[:20]])
    if len(bad): print(b[bad[:5]], ref[bad[:5]])
