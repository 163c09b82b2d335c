"""Multi-GPU plumbing (one process per GPU, torch.distributed): row slabs, the coefficient
halo, and the final reductions.

Rows are independent: rank r owns the contiguous x-lines of ``api.slab_rows`` (a
range along the slowest axes) and assembles them with no data-path collective.  The only exchanges are
* ``exchange_halo`` -- for a user-supplied (not seeded) vertex field distributed by owned
  planes, the p planes below and the 1 plane above a rank's rows (NCCL P2P over NVLink;
  a seeded field is instead regenerated per rank by ``wgq_generate_grid``), and
* ``exchange_u_halo`` -- for the matrix-free product (``wgq_apply``), the rows of u in the
  p planes below and above a rank's slab (the columns its rows touch), P2P from the
  neighbours, and
* ``reduce_checks`` / ``max_time`` -- checksum, norms and the max-over-ranks step time.
Everything here is host logic; the arithmetic of the method stays in libwgq.
"""
import torch
import torch.distributed as dist

from . import api

_p2p_ready = set()


def _p2p(sends, recvs, group=None):
    """Post the point-to-point transfers of one exchange together: ``sends`` / ``recvs`` are
    lists of (tensor, peer).  One ``batch_isend_irecv`` (a ncclGroupStart/End group under
    NCCL) so that two ranks sending to each other cannot deadlock on the per-pair NCCL stream
    the way one-at-a-time isend/irecv can.  Under gloo (host transport) CUDA tensors are staged
    through host memory.  The first P2P call on a group must be made by all its ranks (NCCL
    communicator setup), so a barrier precedes it once per group."""
    torch.cuda.nvtx.range_push("wgq halo exchange")
    try:
        _p2p_inner(sends, recvs, group)
    finally:
        torch.cuda.nvtx.range_pop()


def _p2p_inner(sends, recvs, group):
    key = id(group)
    if key not in _p2p_ready:
        dist.barrier(group=group)
        _p2p_ready.add(key)
    host = dist.get_backend(group) == "gloo"
    staged = []
    ops = []
    for t, peer in sends:
        src = t.cpu() if host and t.is_cuda else t.contiguous()
        ops.append(dist.P2POp(dist.isend, src, peer, group))
    for t, peer in recvs:
        dst = torch.empty(t.shape, dtype=t.dtype) if host and t.is_cuda else t
        staged.append((t, dst))
        ops.append(dist.P2POp(dist.irecv, dst, peer, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    for t, dst in staged:
        if dst is not t:
            t.copy_(dst)


def owned_vertex_planes(n, N, dim, rank, world):
    """Vertex planes [v0, v1) of the slowest axis a rank owns when a user field is
    distributed alongside the row slabs (row planes [z0, z1) clipped to [0, n+1))."""
    plane_rows = N ** (dim - 1)
    b, e = api.slab_rows(N, dim, rank, world)
    z0, z1 = b // plane_rows, e // plane_rows
    return min(z0, n + 1), min(z1, n + 1)


def needed_vertex_planes(p, n, N, dim, rank, world):
    """Vertex planes [lo, hi] touched by the rank's rows: [max(0, z0-p), min(n, z1)]."""
    plane_rows = N ** (dim - 1)
    b, e = api.slab_rows(N, dim, rank, world)
    if e <= b:
        return 0, -1
    z0, z1 = b // plane_rows, (e - 1) // plane_rows
    return max(0, z0 - p), min(n, z1 + 1)


def exchange_halo(owned, p, n, N, dim, group=None):
    """Given this rank's owned vertex planes ``owned`` ([v1-v0, ...] tensor), return the
    planes [lo, hi] its rows need (owned planes plus halo from the neighbours) and lo.
    Point-to-point sends of whole planes; works with NCCL (device tensors) and gloo."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    own = [owned_vertex_planes(n, N, dim, r, world) for r in range(world)]
    need = [needed_vertex_planes(p, n, N, dim, r, world) for r in range(world)]
    lo, hi = need[rank]
    plane_shape = owned.shape[1:]
    out = torch.empty((max(hi - lo + 1, 0),) + tuple(plane_shape), dtype=owned.dtype, device=owned.device)
    sends, recvs = [], []
    # receive: planes of [lo, hi] owned by other ranks
    for src in range(world):
        a, b = max(lo, own[src][0]), min(hi + 1, own[src][1])
        if a >= b:
            continue
        if src == rank:
            out[a - lo:b - lo] = owned[a - own[rank][0]:b - own[rank][0]]
        else:
            recvs.append((out[a - lo:b - lo], _peer(src, group)))
    # send: my owned planes other ranks need
    for dst in range(world):
        if dst == rank:
            continue
        dlo, dhi = need[dst]
        a, b = max(dlo, own[rank][0]), min(dhi + 1, own[rank][1])
        if a >= b:
            continue
        sends.append((owned[a - own[rank][0]:b - own[rank][0]], _peer(dst, group)))
    _p2p(sends, recvs, group)
    return out, lo


def needed_u_rows(p, N, dim, rank, world):
    """Rows [lo, hi) of u that the rank's rows touch: the slowest-axis planes of its slab
    +- p (clipped), as global row ids."""
    plane_rows = N ** (dim - 1)
    b, e = api.slab_rows(N, dim, rank, world)
    if e <= b:
        return 0, 0
    if dim == 1:
        return max(0, b - p), min(N, e + p)
    z0, z1 = b // plane_rows, (e - 1) // plane_rows
    return max(0, z0 - p) * plane_rows, min(N, z1 + p + 1) * plane_rows


def exchange_u_halo(u_owned, p, N, dim, group=None):
    """Given this rank's slab of u (its own rows, flat), return (u_ext, u_row0): u over the rows
    its rows touch (own rows plus the halo from the neighbours) and the global row id of
    u_ext[0], ready for ``wgq_apply``.  P2P sends of contiguous row ranges."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    own = [api.slab_rows(N, dim, r, world) for r in range(world)]
    need = [needed_u_rows(p, N, dim, r, world) for r in range(world)]
    lo, hi = need[rank]
    out = torch.empty(max(hi - lo, 0), dtype=u_owned.dtype, device=u_owned.device)
    sends, recvs = [], []
    for src in range(world):
        a, b = max(lo, own[src][0]), min(hi, own[src][1])
        if a >= b:
            continue
        if src == rank:
            out[a - lo:b - lo] = u_owned[a - own[rank][0]:b - own[rank][0]]
        else:
            recvs.append((out[a - lo:b - lo], _peer(src, group)))
    for dst in range(world):
        if dst == rank:
            continue
        a, b = max(need[dst][0], own[rank][0]), min(need[dst][1], own[rank][1])
        if a >= b:
            continue
        sends.append((u_owned[a - own[rank][0]:b - own[rank][0]], _peer(dst, group)))
    _p2p(sends, recvs, group)
    return out, lo


def apply_distributed(rules, coeff, u_owned, kinds=("mass", "stiffness"), group=None, stream=None):
    """Matrix-free y = A u on this rank's slab: halo exchange of u, then ``wgq_apply``."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    b, e = api.slab_rows(rules.N, rules.dim, rank, world)
    u_ext, u0 = exchange_u_halo(u_owned, rules.p, rules.N, rules.dim, group)
    return api.apply(rules, coeff, u_ext, kinds, b, e, u_row0=u0, stream=stream)


def _peer(r, group):
    """Global rank of group rank r (P2POp takes global ranks)."""
    return r if group is None else dist.get_global_rank(group, r)


def reduce_checks(local, group=None):
    """Sum per-rank (hash, sum, sum of squares) checks: the uint64 hash as a wrapping int64
    sum (== sum mod 2^64), the FP64 sums as doubles."""
    h = local[0:1].view(torch.int64).clone()
    s = local[1:3].view(torch.float64).clone()
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    return int(h.item()) & (2 ** 64 - 1), float(s[0].item()), float(s[1].item())


def max_time(ms, device, group=None):
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
