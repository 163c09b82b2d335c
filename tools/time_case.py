"""Device-time a config's assembly (kernel experiments; not the bench contract).

    python tools/time_case.py --config C5 [--n 256] [--reps 5] [--dbg 0,1,2]

Prints ms per launch (CUDA events, best and median of reps, L2 flushed between reps) and
the achieved algorithmic GB/s, for each WGQ_LINE_DBG mode listed (profiling switches of the
line kernel: 1 = skip compute, 2 = skip stores).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1710_01048_b200 import api, wgq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--dbg", default="0")
ap.add_argument("--ld", type=int, default=None)
ap.add_argument("--op", default="assemble", choices=["assemble", "load", "apply", "csr"])
ap.add_argument("--slab", default=None, help="r/W: only rank r's rows of a W-way line-granular split (assemble)")
a = ap.parse_args()
cfg = inputs.config(a.config, a.n)
rules = wgq.Rules(cfg["p"], cfg["n"], cfg["dim"])
rb, re_ = 0, rules.n_rows
if a.slab:
    r_, w_ = map(int, a.slab.split("/"))
    rb, re_ = api.slab_rows(rules.N, rules.dim, r_, w_)
grid, plane0 = (None, 0)
if cfg["coeff"]["kind"] == "grid":
    grid, plane0 = api.make_grid(rules, cfg["coeff"]["seed"], cfg["coeff"]["sigma"], rb, re_)
coef = api.coefficient(inputs.coefficient(cfg["coeff"], cfg["dim"]), grid, plane0)
out = {k: api.alloc_ell(rules, rb, re_, a.ld) for k in cfg["kinds"]} if a.op == "assemble" else None
u = torch.randn(rules.n_rows, dtype=torch.float64, device="cuda") if a.op == "apply" else None
if a.op == "csr":
    nnz = wgq.wgq_nnz(rules, 0, rules.n_rows)
    row_ptr = torch.empty(rules.n_rows + 1, dtype=torch.int64, device="cuda")
    col_idx = torch.empty(nnz, dtype=torch.int32, device="cuda")
    wgq.wgq_csr_structure(rules, 0, rules.n_rows, row_ptr, col_idx)
    vals = {k: torch.empty(nnz, dtype=torch.float64, device="cuda") for k in cfg["kinds"]}
    descs = {k: wgq.make_out(vals[k], 0, rules.n_rows, ld=0, layout=wgq.WGQ_CSR, row_ptr=row_ptr) for k in cfg["kinds"]}
bvec = torch.empty(rules.n_rows, dtype=torch.float64, device="cuda") if a.op == "load" else None


def run():
    if a.op == "assemble":
        api.assemble(rules, coef, cfg["kinds"], rb, re_, out=out)
    elif a.op == "load":
        api.assemble_load(rules, coef, out=bvec)
    elif a.op == "csr":
        if len(cfg["kinds"]) == 2:
            wgq.wgq_assemble_mass_stiffness(rules, coef, descs["mass"], descs["stiffness"])
        else:
            wgq.wgq_assemble_mass(rules, coef, descs["mass"])
    else:
        api.apply(rules, coef, u, cfg["kinds"])
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
alg = ((re_ - rb) * rules.stencil * 8 * len(cfg["kinds"]) if a.op == "assemble" else
       wgq.wgq_nnz(rules, 0, rules.n_rows) * 8 * len(cfg["kinds"]) if a.op == "csr" else rules.n_rows * 8)
res = {}
for mode in a.dbg.split(","):
    os.environ["WGQ_LINE_DBG"] = mode
    run()
    ts = []
    for _ in range(a.reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    res[mode] = {"best_ms": round(ts[0], 4), "median_ms": round(ts[len(ts) // 2], 4),
                 "GBs": round(alg / ts[0] / 1e6, 1), "all": [round(x, 3) for x in ts]}
print(json.dumps({"config": cfg["name"], "op": a.op, "n": cfg["n"], "rows": re_ - rb, "slab": a.slab, "modes": res}))
