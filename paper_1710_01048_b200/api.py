"""Tensor-level convenience layer over the C-ABI (allocation, slabs, streams).

Everything numerical runs in libwgq's CUDA kernels; this module only sizes buffers,
builds descriptors and picks row ranges.  Row slabs follow the z-slab (3D) / y-slab (2D)
partition of SURVEY §8(e): contiguous ranges of the slowest row index.
"""
import torch

from . import wgq


def slab_rows(N, dim, rank, world):
    """N: rows per direction (an int, or per-direction sizes for an anisotropic mesh)."""
    Ns = [int(N)] * dim if not hasattr(N, "__len__") else [int(v) for v in N]
    return _slab_rows(Ns, dim, rank, world)


def _slab_rows(Ns, dim, rank, world):
    """Row range [b, e) of rank's slab: contiguous rows along the slowest axes, split into
    whole x-lines (N rows; single rows in 1D) as evenly as possible (the first lines % world
    ranks get one more line).  Line granularity keeps the ranks within one line (0.01 % at C5
    on 8 GPUs) instead of one z-plane (1.9 %) of each other; a slab may start or end inside a
    z-plane, which every kernel and the halo logic handle."""
    unit = Ns[0] if dim >= 2 else 1
    total = 1
    for v in Ns[:dim]:
        total *= v
    units = total // unit
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return u0 * unit, u1 * unit


def _ns(rules):
    return list(getattr(rules, "ns", [rules.n] * rules.dim)), list(getattr(rules, "Ns", [rules.N] * rules.dim))


def grid_planes_for(rules, row_begin, row_end):
    """Vertex planes [lo, hi] of the slowest axis touched by rows [row_begin, row_end)."""
    ns, Ns = _ns(rules)
    plane_rows = 1
    for v in Ns[:rules.dim - 1]:
        plane_rows *= v
    z0 = row_begin // plane_rows
    z1 = (row_end - 1) // plane_rows
    return max(0, z0 - rules.p), min(ns[rules.dim - 1], z1 + 1)


def make_grid(rules, seed, sigma, row_begin, row_end, device=None, stream=None):
    """Device-generated lognormal vertex slab covering rows [row_begin, row_end):
    returns (grid tensor, plane0)."""
    dim = rules.dim
    ns, _ = _ns(rules)
    lo, hi = (0, ns[0]) if dim == 1 else grid_planes_for(rules, row_begin, row_end)
    planes = hi - lo + 1
    shape = {1: (ns[0] + 1,), 2: (planes, ns[0] + 1), 3: (planes, ns[1] + 1, ns[0] + 1)}[dim]
    g = torch.empty(shape, dtype=torch.float64, device=device or "cuda")
    wgq.wgq_generate_grid(ns, dim, seed, sigma, lo, planes, g, stream)
    return g, lo


def coefficient(desc, grid=None, plane0=0):
    return wgq.make_coeff(desc, grid, plane0)


def alloc_ell(rules, row_begin, row_end, ld=None, device=None):
    ld = ld or rules.stencil
    return torch.empty((row_end - row_begin, ld), dtype=torch.float64, device=device or "cuda")


def assemble(rules, coeff, kinds=("mass", "stiffness"), row_begin=0, row_end=None, ld=None, out=None, stream=None):
    """Assemble rows [row_begin, row_end) in ELL layout; returns {'mass': T, 'stiffness': T}."""
    if row_end is None:
        row_end = rules.n_rows
    out = dict(out or {})
    for k in kinds:
        if k not in out:
            out[k] = alloc_ell(rules, row_begin, row_end, ld)
    descs = {k: wgq.make_out(out[k], row_begin, row_end, ld=out[k].shape[1]) for k in kinds}
    if "mass" in kinds and "stiffness" in kinds:
        wgq.wgq_assemble_mass_stiffness(rules, coeff, descs["mass"], descs["stiffness"], stream)
    elif "mass" in kinds:
        wgq.wgq_assemble_mass(rules, coeff, descs["mass"], stream)
    else:
        wgq.wgq_assemble_stiffness(rules, coeff, descs["stiffness"], stream)
    return out


def assemble_csr(rules, coeff, kinds=("mass", "stiffness"), row_begin=0, row_end=None, stream=None):
    """CSR assembly: returns (row_ptr int64, col_idx int32, {'mass': values, ...})."""
    if row_end is None:
        row_end = rules.n_rows
    nnz = wgq.wgq_nnz(rules, row_begin, row_end)
    row_ptr = torch.empty(row_end - row_begin + 1, dtype=torch.int64, device="cuda")
    col_idx = torch.empty(nnz, dtype=torch.int32, device="cuda")
    wgq.wgq_csr_structure(rules, row_begin, row_end, row_ptr, col_idx, stream)
    vals = {k: torch.empty(nnz, dtype=torch.float64, device="cuda") for k in kinds}
    descs = {k: wgq.make_out(vals[k], row_begin, row_end, ld=0, layout=wgq.WGQ_CSR, row_ptr=row_ptr) for k in kinds}
    if "mass" in kinds and "stiffness" in kinds:
        wgq.wgq_assemble_mass_stiffness(rules, coeff, descs["mass"], descs["stiffness"], stream)
    elif "mass" in kinds:
        wgq.wgq_assemble_mass(rules, coeff, descs["mass"], stream)
    else:
        wgq.wgq_assemble_stiffness(rules, coeff, descs["stiffness"], stream)
    return row_ptr, col_idx, vals


def assemble_load(rules, f, row_begin=0, row_end=None, out=None, stream=None):
    """Load vector b_i = int f B_i by the rows' mass rules (eq:Load) for rows [row_begin, row_end)."""
    if row_end is None:
        row_end = rules.n_rows
    b = out if out is not None else torch.empty(row_end - row_begin, dtype=torch.float64, device="cuda")
    wgq.wgq_assemble_load(rules, f, row_begin, row_end, b, stream)
    return b


def apply(rules, coeff, u, kinds=("mass", "stiffness"), row_begin=0, row_end=None, u_row0=0, stream=None):
    """Matrix-free y = A u for the rows [row_begin, row_end) (u: global rows from u_row0)."""
    if row_end is None:
        row_end = rules.n_rows
    rows = row_end - row_begin
    y = {k: torch.empty(rows, dtype=torch.float64, device="cuda") for k in kinds}
    wgq.wgq_apply(rules, coeff, u, u_row0, row_begin, row_end, y.get("mass"), y.get("stiffness"), stream)
    return y


def rules_json(rules):
    """The handle's unit-spacing rules as JSON: a list of
    {kind, degree, class, nodes[], weights[], residual_max}, nodes / weights with 17
    significant digits; class 0..p-1 = left boundary weight j, "interior" = the shift-invariant rule."""
    import json
    out = []
    for kind, kc in (("mass", wgq.WGQ_MASS), ("stiffness", wgq.WGQ_STIFFNESS)):
        for cls in range(rules.p + 1):
            tau, om, res = wgq.wgq_rules_query(rules, cls, kc)
            out.append({"kind": kind, "degree": rules.p, "class": "interior" if cls == rules.p else cls,
                        "nodes": [float(f"{x:.17g}") for x in tau], "weights": [float(f"{w:.17g}") for w in om],
                        "residual_max": float(res)})
    return json.dumps(out, indent=1)
