"""Command-line front end of libwgq (the C-ABI error codes mapped to exit codes).

    python -m paper_1710_01048_b200 derive-rules --degree 3 [--kind mass|stiffness] [--boundary gauss|gl] [--out rules.json]
    python -m paper_1710_01048_b200 counts --degree 2 --dim 2 --mesh 100
    python -m paper_1710_01048_b200 assemble --degree 3 --dim 3 --mesh 64 [--coef grid|const|trig|fourier]
        (--mesh 64,64,48: one element count per direction)
                                      [--kinds mass,stiffness] [--layout ell|csr] [--mtx out_prefix]
    python -m paper_1710_01048_b200 eigen --degree 2 --dim 1 --mesh 1000 [--count 10]

Exit codes: 0 success, 2 validation failure (a rule residual above tolerance),
3 solver failure (WGQ_ENOCONV), 4 configuration error (bad arguments, WGQ_EINVAL /
WGQ_EUNSUPPORTED / WGQ_ERANGE).  Numbers are printed with 17 significant digits.  Every
computation runs in libwgq; this module only parses arguments and writes files.
"""
import argparse
import json
import sys

EXIT_OK, EXIT_VALIDATION, EXIT_SOLVER, EXIT_CONFIG = 0, 2, 3, 4


def _exit_for(err):
    from . import wgq
    if err.code == wgq.WGQ_ENOCONV:
        return EXIT_SOLVER
    return EXIT_CONFIG


def cmd_derive_rules(a):
    from . import api, wgq
    r = wgq.Rules(a.degree, max(a.degree + 1, 8), 1, wgq.WGQ_BND_GL if a.boundary == "gl" else wgq.WGQ_BND_GAUSS)
    doc = [e for e in json.loads(api.rules_json(r)) if a.kind in (None, e["kind"])]
    text = json.dumps(doc, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text + "\n")
    else:
        print(text)
    worst = max(e["residual_max"] for e in doc)
    return EXIT_OK if worst <= a.tol else EXIT_VALIDATION


def cmd_counts(a):
    from . import wgq
    r = wgq.Rules(a.degree, a.mesh, a.dim)
    out = {}
    for kind, kc in (("mass", wgq.WGQ_MASS), ("stiffness", wgq.WGQ_STIFFNESS)):
        g, c = wgq.wgq_eval_counts(r, kc)
        out[kind] = {"gaussian": g, "newton_cotes": c, "ratio": float(f"{c / g:.17g}")}
    print(json.dumps(out, indent=1))
    return EXIT_OK


def _coef(a, rules):
    from . import api
    import inputs
    if a.coef == "grid":
        grid, plane0 = api.make_grid(rules, inputs.SEED, 0.5, 0, rules.n_rows)
        return api.coefficient({"kind": "grid"}, grid, plane0)
    if a.coef == "const":
        return api.coefficient({"kind": "const", "c0": 1.0})
    if a.coef == "trig":
        return api.coefficient({"kind": "trig_sep", "c0": 1.0, "amp": 0.5, "trig": ("sin", "cos", "sin")[:a.dim],
                                "wavenum": (1, 1, 1)[:a.dim]})
    return api.coefficient(inputs.coefficient({"kind": "fourier_logn", "seed": inputs.SEED, "n_modes": 8,
                                               "amp": 0.3}, a.dim))


def _write_mtx(path, N, rows, cols, vals):
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{N} {N} {len(vals)}\n")
        for r, c, v in zip(rows, cols, vals):
            f.write(f"{r + 1} {c + 1} {v:.17g}\n")


def cmd_assemble(a):
    import numpy as np
    import torch

    from . import api, wgq
    kinds = tuple(k.strip() for k in a.kinds.split(","))
    if any(k not in ("mass", "stiffness") for k in kinds):
        print("kinds must be mass and/or stiffness", file=sys.stderr)
        return EXIT_CONFIG
    rules = wgq.Rules(a.degree, a.mesh if len(a.mesh) > 1 else a.mesh[0], a.dim)
    c = _coef(a, rules)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if a.layout == "ell":
        out = api.assemble(rules, c, kinds)                   # warm-up (tables)
        e0.record()
        out = api.assemble(rules, c, kinds, out=out)
        e1.record()
    else:
        row_ptr, col_idx, out = api.assemble_csr(rules, c, kinds)
        e0.record()
        row_ptr, col_idx, out = api.assemble_csr(rules, c, kinds)
        e1.record()
    torch.cuda.synchronize()
    nnz = wgq.wgq_nnz(rules, 0, rules.n_rows)
    report = {"rows": rules.n_rows, "nnz_per_matrix": nnz, "ms": float(f"{e0.elapsed_time(e1):.17g}"),
              "layout": a.layout, "kinds": list(kinds)}
    if a.mtx:
        if a.layout == "ell":
            row_ptr, col_idx, out = api.assemble_csr(rules, c, kinds)
            torch.cuda.synchronize()
        rp, ci = row_ptr.cpu().numpy(), col_idx.cpu().numpy()
        rows = np.repeat(np.arange(rules.n_rows), np.diff(rp))
        for k in kinds:
            _write_mtx(f"{a.mtx}_{k}.mtx", rules.n_rows, rows, ci, out[k].cpu().numpy())
        report["files"] = [f"{a.mtx}_{k}.mtx" for k in kinds]
    print(json.dumps(report, indent=1))
    return EXIT_OK


def cmd_eigen(a):
    from . import api, eigen, wgq
    rules = wgq.Rules(a.degree, a.mesh, a.dim)
    lam = eigen.spectrum(rules, api.coefficient({"kind": "const", "c0": 1.0})).cpu().tolist()
    count = min(a.count, len(lam))
    ex = eigen.exact_eigenvalues(a.dim, count)
    print(json.dumps({"dofs": len(lam), "exact": ex, "discrete": lam[:count],
                      "rel_err": [float(f"{lam[k] / ex[k] - 1:.17g}") for k in range(count)]}, indent=1))
    return EXIT_OK


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1710_01048_b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="cmd", required=True)
    d = sub.add_parser("derive-rules", help="build and export the weighted Gaussian rules (JSON)")
    d.add_argument("--degree", type=int, required=True)
    d.add_argument("--kind", choices=["mass", "stiffness"], default=None)
    d.add_argument("--boundary", choices=["gauss", "gl"], default="gauss")
    d.add_argument("--tol", type=float, default=1e-12, help="residual tolerance (exit 2 above it)")
    d.add_argument("--out", default=None)
    c = sub.add_parser("counts", help="basis-evaluation counts, Gaussian vs Newton-Cotes (E3)")
    c.add_argument("--degree", type=int, required=True)
    c.add_argument("--dim", type=int, default=2)
    c.add_argument("--mesh", type=int, default=100)
    s = sub.add_parser("assemble", help="assemble M and/or K on the GPU")
    s.add_argument("--degree", type=int, required=True)
    s.add_argument("--dim", type=int, required=True)
    s.add_argument("--mesh", type=lambda v: [int(x) for x in v.split(",")], required=True,
                   help="elements per direction: one count, or one per direction (e.g. 64,64,48)")
    s.add_argument("--coef", choices=["grid", "const", "trig", "fourier"], default="const")
    s.add_argument("--kinds", default="mass,stiffness")
    s.add_argument("--layout", choices=["ell", "csr"], default="ell")
    s.add_argument("--mtx", default=None, help="write MatrixMarket files <prefix>_<kind>.mtx")
    e = sub.add_parser("eigen", help="Dirichlet Laplacian spectrum from the assembled M, K (E1/E2)")
    e.add_argument("--degree", type=int, required=True)
    e.add_argument("--dim", type=int, default=1)
    e.add_argument("--mesh", type=int, required=True)
    e.add_argument("--count", type=int, default=10)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_CONFIG if e.code else EXIT_OK
    from . import wgq
    try:
        return {"derive-rules": cmd_derive_rules, "counts": cmd_counts, "assemble": cmd_assemble, "eigen": cmd_eigen}[a.cmd](a)
    except wgq.WgqError as err:
        print(str(err), file=sys.stderr)
        return _exit_for(err)


if __name__ == "__main__":
    sys.exit(main())
