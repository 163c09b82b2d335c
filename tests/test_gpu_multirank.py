"""The N > 1 path on the GPU box, self-verifying: rows are independent
(the row-wise local quadrature mask), so a z-slab split must reproduce the
one-rank result exactly.

* bench.py under torchrun with 2 ranks (WGQ_BENCH_FUNCTIONAL=1: both ranks on cuda:0, gloo for
  the reductions -- a functional check of the multi-rank code path, never a measurement; the
  ranks' kernels do not wait on one another) prints the same checksum hash as the 1-rank run
  and counts the whole mesh's nonzeros.
* the halo exchanges of dist.py with CUDA tensors (2 ranks, gloo staging through the host)
  deliver exactly the planes / rows a rank needs, and the distributed matrix-free product
  equals the one-rank product.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _bench(args, ranks=1, env=None):
    e = dict(os.environ, **(env or {}))
    if ranks == 1:
        cmd = [sys.executable, "bench.py"] + args
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", str(ranks)] + args
    r = subprocess.run(cmd, cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("config,elems", [("C5", 48), ("C3", 64)])
def test_bench_two_ranks_reproduce_one_rank_checksum(config, elems):
    from paper_1710_01048_b200 import wgq
    common = ["--config", config, "--elems", str(elems), "--no-e2e", "--no-extras", "--no-cpu", "--steps", "3",
              "--warmup", "3"]
    one = _bench(common)
    two = _bench(common, ranks=2, env={"WGQ_BENCH_FUNCTIONAL": "1"})
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    for k in one["checksum"]:
        assert two["checksum"][k]["hash"] == one["checksum"][k]["hash"], k
        assert two["checksum"][k]["sum"] == pytest.approx(one["checksum"][k]["sum"], rel=1e-12)
    import inputs
    cfg = inputs.config(config, elems)
    rules = wgq.Rules(cfg["p"], cfg["n"], cfg["dim"])
    assert one["nnz_per_step"] == two["nnz_per_step"] == wgq.wgq_nnz(rules, 0, rules.n_rows) * len(cfg["kinds"])


def _halo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    import inputs
    from paper_1710_01048_b200 import api, wgq
    from paper_1710_01048_b200 import dist as wdist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, n, d = 3, 9, 3
        rules = wgq.Rules(p, n, d)
        N = rules.N
        full = torch.from_numpy(inputs.lognormal_grid(n, seed=17, dim=d)).cuda()
        v0, v1 = wdist.owned_vertex_planes(n, N, d, rank, world)
        got, lo = wdist.exchange_halo(full[v0:v1].clone(), p, n, N, d)
        lo2, hi2 = wdist.needed_vertex_planes(p, n, N, d, rank, world)
        ok_grid = got.is_cuda and lo == lo2 and torch.equal(got, full[lo2:hi2 + 1])
        # the distributed matrix-free product with the exchanged (user) grid slab
        coef = api.coefficient({"kind": "grid"}, got, lo)
        u = torch.from_numpy(np.random.default_rng(5).standard_normal(N ** d)).cuda()
        b, e = api.slab_rows(N, d, rank, world)
        y = wdist.apply_distributed(rules, coef, u[b:e].clone())
        torch.cuda.synchronize()
        q.put((rank, bool(ok_grid), b, e, {k: v.cpu().numpy() for k, v in y.items()}))
    finally:
        dist.destroy_process_group()


def test_halo_exchange_and_distributed_apply_with_cuda_tensors():
    import torch.multiprocessing as mp

    import inputs
    from paper_1710_01048_b200 import api, wgq
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p, n, d = 3, 9, 3
    rules = wgq.Rules(p, n, d)
    N = rules.N
    grid = torch.from_numpy(inputs.lognormal_grid(n, seed=17, dim=d)).cuda()
    u = torch.from_numpy(np.random.default_rng(5).standard_normal(N ** d)).cuda()
    y1 = api.apply(rules, api.coefficient({"kind": "grid"}, grid, 0), u)
    torch.cuda.synchronize()
    for rank, ok_grid, b, e, y in res:
        assert ok_grid, rank
        for k in ("mass", "stiffness"):
            assert np.array_equal(y[k], y1[k].cpu().numpy()[b:e]), (rank, k)
