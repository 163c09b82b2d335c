"""Run a few assemblies of a config for profiling (ncu / compute-sanitizer targets).

    python tools/profile_case.py --config C5 --n 128 --launches 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1710_01048_b200 import api, wgq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--launches", type=int, default=2)
ap.add_argument("--ld", type=int, default=None)
a = ap.parse_args()
cfg = inputs.config(a.config, a.n)
rules = wgq.Rules(cfg["p"], cfg["n"], cfg["dim"])
grid, plane0 = (None, 0)
if cfg["coeff"]["kind"] == "grid":
    grid, plane0 = api.make_grid(rules, cfg["coeff"]["seed"], cfg["coeff"]["sigma"], 0, rules.n_rows)
coef = api.coefficient(inputs.coefficient(cfg["coeff"], cfg["dim"]), grid, plane0)
out = {k: api.alloc_ell(rules, 0, rules.n_rows, a.ld) for k in cfg["kinds"]}
for _ in range(a.launches):
    api.assemble(rules, coef, cfg["kinds"], out=out)
torch.cuda.synchronize()
print("ok", cfg["name"], cfg["n"], rules.n_rows)
