"""Multi-process host logic of the multi-GPU path on CPU (gloo, world_size 2 and 3).

The kernels never run here: these tests cover the slab partition, the vertex-plane halo
exchange for a user-supplied field and the cross-rank reductions that bench.py and a
multi-GPU user rely on.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
from paper_1710_01048_b200 import api, dist as wdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, n, dim, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = n + p
        full = torch.from_numpy(inputs.lognormal_grid(n, seed=13, dim=dim))
        v0, v1 = wdist.owned_vertex_planes(n, N, dim, rank, world)
        owned = full[v0:v1].clone()
        got, lo = wdist.exchange_halo(owned, p, n, N, dim)
        lo2, hi2 = wdist.needed_vertex_planes(p, n, N, dim, rank, world)
        ok_halo = lo == lo2 and torch.equal(got, full[lo2:hi2 + 1])
        # u halo for the matrix-free product: own planes +- p from the neighbours
        u_full = torch.arange(N ** dim, dtype=torch.float64) * 0.5 + 3.0
        b, e = api.slab_rows(N, dim, rank, world)
        u_ext, u0 = wdist.exchange_u_halo(u_full[b:e].clone(), p, N, dim)
        plane_rows = N ** (dim - 1)
        ulo, uhi = wdist.needed_u_rows(p, N, dim, rank, world)
        ok_u = (u0 == ulo and torch.equal(u_ext, u_full[ulo:uhi])
                and (e <= b or (u0 <= max(0, b // plane_rows - p) * plane_rows
                                and u0 + u_ext.numel() >= min(N, (e - 1) // plane_rows + p + 1) * plane_rows)))
        ok_halo = ok_halo and ok_u
        # reductions: hash wraps mod 2^64, sums add
        local = torch.zeros(3, dtype=torch.float64)
        local[0:1].view(torch.int64)[0] = (2 ** 63 - 5) if rank == 0 else 11
        local[1] = rank + 1.0
        local[2] = (rank + 1.0) ** 2
        h, s1, s2 = wdist.reduce_checks(local)
        t = wdist.max_time(10.0 * (rank + 1), "cpu")
        q.put((rank, ok_halo, h, s1, s2, t, api.slab_rows(N, dim, rank, world)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,p,n,dim", [(2, 3, 8, 3), (3, 2, 5, 3), (2, 3, 10, 2), (3, 3, 4, 3)])
def test_halo_reductions_and_slabs(world, p, n, dim):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, n, dim, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    N = n + p
    slabs = [r[6] for r in res]
    assert slabs[0][0] == 0 and slabs[-1][1] == N ** dim
    assert all(slabs[i][1] == slabs[i + 1][0] for i in range(world - 1))
    sizes = [e - b for b, e in slabs]
    assert max(sizes) - min(sizes) <= N                        # line-granular balance
    assert all(b % N == 0 for b, _ in slabs)                   # whole x-lines
    for rank, ok_halo, h, s1, s2, t, _ in res:
        assert ok_halo, rank
        expect_h = ((2 ** 63 - 5) + 11 * (world - 1)) % 2 ** 64
        assert h == expect_h
        assert s1 == sum(range(1, world + 1)) and s2 == sum(k * k for k in range(1, world + 1))
        assert t == 10.0 * world


def test_grid_planes_cover_every_row():
    """The device grid slab a rank generates covers every element its rows touch."""
    for p, n in ((2, 9), (3, 12)):
        N = n + p
        rules = type("R", (), {"N": N, "dim": 3, "p": p, "n": n})
        for world in (1, 2, 5, 8):
            for r in range(world):
                b, e = api.slab_rows(N, 3, r, world)
                if e <= b:
                    continue
                lo, hi = api.grid_planes_for(rules, b, e)
                z0, z1 = b // (N * N), (e - 1) // (N * N)
                for z in (z0, z1):
                    elems = range(max(0, z - p), min(n - 1, z) + 1)
                    assert all(lo <= el and el + 1 <= hi for el in elems)
