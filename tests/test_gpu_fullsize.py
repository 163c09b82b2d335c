"""Full-size parity at BASELINE.json's sizes, in the launch configuration bench.py times.

Each config is assembled on the GPU exactly as bench.py does (api.assemble over the whole
mesh, device-generated GRID field for C5); the oracle recomputes a sample of rows one by one
(every boundary / near-boundary row class plus random interior rows) and the GPU rows must
match them (R12).  Properties that hold at any size are checked on ALL rows on the device:
(K 1)_i = 0 (P9) and the 8-slab z-partition of C5 reproduces the one-GPU checksum exactly.
"""
import os

import numpy as np
import pytest

import inputs
from oracle import assemble as oasm

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from parity import compare  # noqa: E402


def sample_rows(p, n, d, count, seed):
    """Row sample covering every class combination: per direction the indices 0..2p+1,
    N-2p-2..N-1 and random interior ones."""
    N = n + p
    rng = np.random.default_rng(seed)
    edge = sorted(set(list(range(0, 2 * p + 2)) + list(range(N - 2 * p - 2, N))))
    rows = set()
    while len(rows) < count:
        idx = []
        for _ in range(d):
            idx.append(int(rng.choice(edge)) if rng.random() < 0.5 else int(rng.integers(0, N)))
        rows.add(sum(idx[a] * N ** a for a in range(d)))
    return np.array(sorted(rows))


def check_rows(gpu_rows, ref, sc, what):
    compare(gpu_rows, ref, what, sc)


def assemble_config(name):
    from paper_1710_01048_b200 import api, wgq
    cfg = inputs.config(name)
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    rules = wgq.Rules(p, n, d)
    desc = inputs.coefficient(cfg["coeff"], d)
    grid, plane0 = (None, 0)
    if desc["kind"] == "grid":
        grid, plane0 = api.make_grid(rules, desc["seed"], desc["sigma"], 0, rules.n_rows)
    out = api.assemble(rules, api.coefficient(desc, grid, plane0), cfg["kinds"])
    torch.cuda.synchronize()
    return cfg, rules, desc, out


@pytest.mark.parametrize("name,count", [("C2", 600), ("C3", 400), ("C4", 500), ("C5", 700)])
def test_full_size_sampled_rows(name, count):
    from paper_1710_01048_b200 import wgq
    cfg, rules, desc, out = assemble_config(name)
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    rows = sample_rows(p, n, d, count, seed=sum(map(ord, name)))
    host_grid = None
    if desc["kind"] == "grid":
        host_grid = inputs.lognormal_grid(n, seed=desc["seed"], sigma=desc["sigma"])
    ref = oasm.assemble_rows(p, n, d, rows, desc, cfg["kinds"], grid=host_grid)
    sc = oasm.assemble_rows(p, n, d, rows, desc, cfg["kinds"], grid=host_grid, absolute=True)
    idx = torch.from_numpy(rows).cuda()
    try:
        for k in cfg["kinds"]:
            check_rows(out[k].index_select(0, idx).cpu().numpy(), ref[k], sc[k], (name, k))
        # every row: (K 1)_i = 0 relative to the row's scale (P9); (M 1)_i > 0
        mom = torch.empty((rules.n_rows, 1 + d), dtype=torch.float64, device="cuda")
        if "stiffness" in cfg["kinds"]:
            wgq.wgq_row_moments(rules, wgq.make_out(out["stiffness"], 0, rules.n_rows), mom)
            worst = 0.0
            for lo in range(0, rules.n_rows, 1 << 22):      # chunked: no 95 GB temporaries
                rowmax = out["stiffness"][lo:lo + (1 << 22)].abs().amax(dim=1)
                worst = max(worst, float((mom[lo:lo + (1 << 22), 0].abs() / rowmax).max()))
            assert worst < 1e-12, worst
        if "mass" in cfg["kinds"]:
            wgq.wgq_row_moments(rules, wgq.make_out(out["mass"], 0, rules.n_rows), mom)
            assert bool((mom[:, 0] > 0).all())
        del mom
    finally:
        out.clear()
        torch.cuda.empty_cache()


def test_c5_slabs_reproduce_one_gpu_checksum():
    """8 z-slabs, each with its own device-generated coefficient slab (as 8 ranks would),
    give exactly the one-GPU checksum (order-independent uint64 hash)."""
    from paper_1710_01048_b200 import api, wgq
    cfg, rules, desc, out = assemble_config("C5")
    N = rules.N
    full = {}
    for k in cfg["kinds"]:
        h = torch.zeros(3, dtype=torch.int64, device="cuda")
        wgq.wgq_checksum(rules, wgq.make_out(out[k], 0, rules.n_rows), h)
        full[k] = int(h[0].item()) & (2 ** 64 - 1)
    out.clear()
    torch.cuda.empty_cache()
    acc = {k: 0 for k in cfg["kinds"]}
    buf = None
    for r in range(8):
        b, e = api.slab_rows(N, 3, r, 8)
        grid, plane0 = api.make_grid(rules, desc["seed"], desc["sigma"], b, e)
        if buf is None:
            buf = {k: api.alloc_ell(rules, 0, e - b + N * N) for k in cfg["kinds"]}
        o = {k: buf[k][:e - b] for k in cfg["kinds"]}
        api.assemble(rules, api.coefficient(desc, grid, plane0), cfg["kinds"], b, e, out=o)
        for k in cfg["kinds"]:
            h = torch.zeros(3, dtype=torch.int64, device="cuda")
            wgq.wgq_checksum(rules, wgq.make_out(o[k], b, e), h)
            acc[k] = (acc[k] + int(h[0].item())) % 2 ** 64
    for k in cfg["kinds"]:
        assert acc[k] == full[k], k


def test_c5_csr_full_size_sampled_rows():
    """C5 in CSR layout at full size (117 GB: values of both matrices, int32 columns, int64
    row pointers): sampled rows' pointers, columns and values against the oracle."""
    from paper_1710_01048_b200 import api, wgq
    cfg = inputs.config("C5")
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    rules = wgq.Rules(p, n, d)
    desc = inputs.coefficient(cfg["coeff"], d)
    grid, plane0 = api.make_grid(rules, desc["seed"], desc["sigma"], 0, rules.n_rows)
    row_ptr, col_idx, vals = api.assemble_csr(rules, api.coefficient(desc, grid, plane0), cfg["kinds"])
    torch.cuda.synchronize()
    try:
        N = n + p
        a1 = np.array([min(i + p, N - 1) - max(i - p, 0) + 1 for i in range(N)], dtype=np.int64)
        total = int(a1.sum()) ** 3
        assert int(row_ptr[-1].item()) == total == wgq.wgq_nnz(rules, 0, rules.n_rows)
        rows = sample_rows(p, n, d, 300, seed=5)
        host_grid = inputs.lognormal_grid(n, seed=desc["seed"], sigma=desc["sigma"])
        ref = oasm.assemble_rows(p, n, d, rows, desc, cfg["kinds"], grid=host_grid)
        sc = oasm.assemble_rows(p, n, d, rows, desc, cfg["kinds"], grid=host_grid, absolute=True)
        # row pointers by brute force over the lexicographic rows before r: planes, lines, rows
        A1 = np.concatenate([[0], np.cumsum(a1)])
        S = int(A1[-1])
        rp = row_ptr.index_select(0, torch.from_numpy(np.concatenate([rows, rows + 1])).cuda()).cpu().numpy()
        got = {k: np.zeros((len(rows), rules.stencil)) for k in cfg["kinds"]}
        for t, r in enumerate(rows):
            i1, i2, i3 = r % N, (r // N) % N, r // (N * N)
            start = A1[i3] * S * S + a1[i3] * (A1[i2] * S + a1[i2] * A1[i1])
            assert rp[t] == start and rp[len(rows) + t] - rp[t] == a1[i1] * a1[i2] * a1[i3]
            cols = oasm.ell_columns(p, n, d, int(r))
            ok = cols >= 0
            assert np.array_equal(col_idx[rp[t]:rp[len(rows) + t]].cpu().numpy(), cols[ok])
            for k in cfg["kinds"]:
                got[k][t, ok] = vals[k][rp[t]:rp[len(rows) + t]].cpu().numpy()
        for k in cfg["kinds"]:
            check_rows(got[k], ref[k], sc[k], ("C5 csr", k))
    finally:
        del row_ptr, col_idx, vals
        torch.cuda.empty_cache()


def test_c5_whole_lines_every_class():
    """SURVEY §8(c) P10 at C5, line-wise: whole x-lines (all 259 x-positions, so every x row
    class and every tile position of the line kernel) on the boundary / near-boundary y and z
    classes and a few seeded interior ones, against the oracle row by row."""
    cfg, rules, desc, out = assemble_config("C5")
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    N = n + p
    rng = np.random.default_rng(10)
    ys = [0, 1, 2, 3, 5, 6, N - 7, N - 4, N - 2, N - 1] + [int(v) for v in rng.integers(2 * p + 2, N - 2 * p - 2, 3)]
    zs = [0, 1, 3, 6, N - 5, N - 1] + [int(v) for v in rng.integers(2 * p + 2, N - 2 * p - 2, 2)]
    lines = [(int(ys[k % len(ys)]), int(zs[k % len(zs)])) for k in range(max(len(ys), len(zs)) * 2)]
    lines = sorted(set(lines))[:24]
    rows = np.concatenate([(z * N + y) * N + np.arange(N) for y, z in lines])
    host_grid = inputs.lognormal_grid(n, seed=desc["seed"], sigma=desc["sigma"])
    try:
        ref = oasm.assemble_rows(p, n, d, rows, desc, cfg["kinds"], grid=host_grid)
        sc = oasm.assemble_rows(p, n, d, rows, desc, cfg["kinds"], grid=host_grid, absolute=True)
        idx = torch.from_numpy(rows).cuda()
        for k in cfg["kinds"]:
            check_rows(out[k].index_select(0, idx).cpu().numpy(), ref[k], sc[k], ("C5 lines", k))
    finally:
        out.clear()
        torch.cuda.empty_cache()


_P9_JOBS = None


def _p9_job(i):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    p, n, d, rows, desc, grid, plane0 = _P9_JOBS[i]
    return oasm.row_weight_sums(p, n, d, rows, desc, grid=grid, plane0=plane0)


def test_c5_full_scale_p9_identities():
    """SURVEY §8(c) P9 at the full C5 size (every entry is integrated exactly):
    on EVERY row of the z-planes {0, 1, 3, 6, N-1} and two seeded interior planes (all row
    classes), the GPU matrices' row moments (M 1, M g^a, K 1, K g^a; wgq_row_moments) equal the
    oracle's weighted sums sum_k W^M, sum_k W^M x^a, 0, sum_k W^{K,a} (oracle.assemble.row_weight_sums,
    from the rules and c alone, on its own vertex-plane slab) to 1e-13 x the row maximum."""
    import multiprocessing as mp

    from paper_1710_01048_b200 import wgq
    global _P9_JOBS
    cfg, rules, desc, out = assemble_config("C5")
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    N = rules.N
    P = N * N
    rng = np.random.default_rng(449)
    planes = [0, 1, 3, 6, N - 1] + sorted(int(z) for z in rng.choice(np.arange(2 * p + 1, N - 2 * p - 1), 2, replace=False))
    try:
        gpu = {}
        for z in planes:
            lo, hi = z * P, (z + 1) * P
            for k in ("mass", "stiffness"):
                m = torch.empty((P, 1 + d), dtype=torch.float64, device="cuda")
                wgq.wgq_row_moments(rules, wgq.make_out(out[k][lo:hi], lo, hi), m)
                gpu[(z, k)] = (m.cpu().numpy(), out[k][lo:hi].abs().amax(dim=1).cpu().numpy())
    finally:
        out.clear()
        torch.cuda.empty_cache()
    jobs, where = [], []
    for z in planes:
        gl, gh = max(0, z - p), min(n, z + 1)
        slab = inputs.lognormal_grid(n, seed=desc["seed"], sigma=desc["sigma"], plane0=gl, planes=gh - gl + 1)
        rows = np.arange(z * P, (z + 1) * P)
        for blk in np.array_split(rows, 24):
            jobs.append((p, n, d, blk, desc, slab, gl))
            where.append((z, blk[0] - z * P, len(blk)))
    _P9_JOBS = jobs
    oasm.tables_1d(p, n)
    with mp.get_context("fork").Pool(os.cpu_count() or 1) as pool:
        res = pool.map(_p9_job, range(len(jobs)), chunksize=1)
    worst = {"M1": 0.0, "Mg": 0.0, "K1": 0.0, "Kg": 0.0}
    for (z, off, cnt), (m1, mx, kx) in zip(where, res):
        mm, sM = gpu[(z, "mass")]
        km, sK = gpu[(z, "stiffness")]
        sl = slice(off, off + cnt)
        worst["M1"] = max(worst["M1"], float(np.max(np.abs(mm[sl, 0] - m1) / sM[sl])))
        worst["K1"] = max(worst["K1"], float(np.max(np.abs(km[sl, 0]) / sK[sl])))
        for a in range(d):
            worst["Mg"] = max(worst["Mg"], float(np.max(np.abs(mm[sl, 1 + a] - mx[:, a]) / sM[sl])))
            worst["Kg"] = max(worst["Kg"], float(np.max(np.abs(km[sl, 1 + a] - kx[:, a]) / sK[sl])))
    print("C5 P9 worst relative to row max:", worst, "planes", planes)
    assert worst["M1"] < 1e-13 and worst["Mg"] < 1e-13 and worst["Kg"] < 1e-13 and worst["K1"] < 1e-12, worst


def test_aniso_c5_sized_sampled_rows():
    """A C5-sized mesh with a different element count per direction (256 x 256 x 192; eq:Gmap3
    P:113-120) through the GRID line kernel, as bench.py's extras time it: sampled rows of every
    class combination against the oracle, and (K 1)_i = 0 on every row."""
    from paper_1710_01048_b200 import api, wgq
    p, n, d = 3, (256, 256, 192), 3
    rules = wgq.Rules(p, n, d)
    Ns = rules.Ns
    g, lo = api.make_grid(rules, inputs.SEED, 0.5, 0, rules.n_rows)
    out = api.assemble(rules, api.coefficient({"kind": "grid"}, g, lo))
    torch.cuda.synchronize()
    try:
        rng = np.random.default_rng(192)
        rows = set()
        while len(rows) < 400:
            idx = []
            for a in range(d):
                edge = list(range(0, 2 * p + 2)) + list(range(Ns[a] - 2 * p - 2, Ns[a]))
                idx.append(int(rng.choice(edge)) if rng.random() < 0.5 else int(rng.integers(0, Ns[a])))
            rows.add(idx[0] + Ns[0] * (idx[1] + Ns[1] * idx[2]))
        rows = np.array(sorted(rows))
        host = inputs.lognormal_grid(n, seed=inputs.SEED, sigma=0.5, dim=3)
        desc = {"kind": "grid"}
        ref = oasm.assemble_rows(p, n, d, rows, desc, grid=host)
        sc = oasm.assemble_rows(p, n, d, rows, desc, grid=host, absolute=True)
        idx_t = torch.from_numpy(rows).cuda()
        for k in ("mass", "stiffness"):
            check_rows(out[k].index_select(0, idx_t).cpu().numpy(), ref[k], sc[k], ("aniso C5", k))
        mom = torch.empty((rules.n_rows, 1 + d), dtype=torch.float64, device="cuda")
        wgq.wgq_row_moments(rules, wgq.make_out(out["stiffness"], 0, rules.n_rows), mom)
        worst = 0.0
        for b in range(0, rules.n_rows, 1 << 22):
            rmax = out["stiffness"][b:b + (1 << 22)].abs().amax(dim=1)
            worst = max(worst, float((mom[b:b + (1 << 22), 0].abs() / rmax).max()))
        assert worst < 1e-12, worst
    finally:
        out.clear()
        torch.cuda.empty_cache()
