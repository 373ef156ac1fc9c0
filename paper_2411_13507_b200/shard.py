"""Row-block sharding of the pair matrix across GPUs and the edge-list gather.

SURVEY.md §8(e): rank g evaluates source rows [floor(V g / G), floor(V (g+1) / G)).
Row blocks preserve global row-major (src, dst) order, so the global CSR is the
rank-ordered concatenation of the per-rank edge blocks; the cut runs locally on
each block and the alive / provenance bytes and counters travel with the edges.
The only exchange step is the gather (NCCL all-gather over NVLink) that hands
rank 0 the whole surviving graph for the shortest-path search.
"""

from __future__ import annotations

import ctypes as C

import numpy as np


def row_block(V: int, rank: int, world: int) -> tuple[int, int]:
    return (V * rank) // world, (V * (rank + 1)) // world


def _coll(t, group=None):
    """The tensor a collective runs on: device tensors as-is for NCCL, host copies for gloo
    (the CPU test backend, which has no CUDA collectives)."""
    import torch.distributed as dist

    if t.is_cuda and dist.get_backend(group) == "gloo":
        return t.cpu()
    return t


def allgather_varlen(t, sizes, group=None):
    """All-gather a 1-D tensor whose length differs per rank; returns the rank-ordered concatenation.

    ``sizes`` is the list of per-rank lengths (already exchanged).  Buffers are padded
    to the largest block so one ``all_gather_into_tensor`` moves everything.
    """
    import torch
    import torch.distributed as dist

    world = len(sizes)
    mx = max(int(s) for s in sizes)
    if mx == 0:
        return torch.zeros(0, dtype=t.dtype, device=t.device)
    pad = torch.zeros(mx, dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t
    pad = _coll(pad, group)
    out = torch.empty(world * mx, dtype=t.dtype, device=pad.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return torch.cat([out[r * mx: r * mx + int(sizes[r])] for r in range(world)]).to(t.device)


def exchange_sizes(n: int, device, group=None) -> list[int]:
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = _coll(torch.tensor([n], dtype=torch.int64, device=device), group)
    out = torch.empty(world, dtype=torch.int64, device=t.device)
    dist.all_gather_into_tensor(out, t, group=group)
    return [int(x) for x in out.tolist()]


def gatherv_to_root(t, sizes, root=0, group=None):
    """Gather a 1-D tensor whose length differs per rank onto ``root`` (rank-ordered
    concatenation there, None elsewhere).  Blocks are padded to the largest one so a
    single ``gather`` moves them (NCCL implements it as grouped send/recv)."""
    import torch
    import torch.distributed as dist

    world = len(sizes)
    mx = max(int(x) for x in sizes)
    me = dist.get_rank(group)
    if mx == 0:
        return torch.zeros(0, dtype=t.dtype, device=t.device) if me == root else None
    pad = torch.zeros(mx, dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t
    pad = _coll(pad, group)
    bufs = [torch.empty_like(pad) for _ in range(world)] if me == root else None
    dist.gather(pad, bufs, dst=root, group=group)
    if me != root:
        return None
    return torch.cat([bufs[r][: int(sizes[r])] for r in range(world)]).to(t.device)


def _export(graph, mask, dev):
    import torch

    from . import _native as nat

    lib = graph._ctx.lib
    E = graph.num_edges
    src = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    dst = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    cost = torch.empty(max(E, 1), dtype=torch.float64, device=dev)
    alive = torch.empty(max(E, 1), dtype=torch.uint8, device=dev)
    prov = torch.empty(max(E, 1), dtype=torch.uint8, device=dev)
    nat.check(lib.bzg_graph_export_device(graph._h, C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
                                          C.c_void_p(cost.data_ptr())))
    nat.check(lib.bzg_mask_export_device(mask._device_handle(), C.c_void_p(alive.data_ptr()),
                                         C.c_void_p(prov.data_ptr())))
    return src[:E], dst[:E], cost[:E], alive[:E], prov[:E]


def _adopt(graph, counters, parts):
    """A new BezierGraph (vertices of ``graph``) + CutMask over the gathered edge blocks."""
    import torch

    from . import _native as nat
    from .graph import BezierGraph, CutMask

    lib = graph._ctx.lib
    s, d, c, a, p = (x.contiguous() for x in parts)
    torch.cuda.current_stream().synchronize()  # libbzg copies on its own stream
    h = C.c_void_p()
    nat.check(lib.bzg_graph_with_edges(graph._h, int(s.numel()), C.c_void_p(s.data_ptr()),
                                       C.c_void_p(d.data_ptr()), C.c_void_p(c.data_ptr()), 1, C.byref(h)))
    g2 = BezierGraph(h, graph._ctx, graph.spec, graph.oracle, graph.seed, graph.sample_bounds, graph._D)
    hm = C.c_void_p()
    nat.check(lib.bzg_mask_from_arrays(graph._ctx.handle, g2._h, C.c_void_p(a.data_ptr()),
                                       C.c_void_p(p.data_ptr()), nat.ptr(counters), 1, C.byref(hm)))
    return g2, CutMask(hm, g2, counters)


def _counters(mask, dev, group, root=None):
    import torch
    import torch.distributed as dist

    cnt = _coll(torch.tensor([mask.pairs_total, mask.pairs_point_hit, mask.pairs_hyperplane, mask.pairs_qp,
                              mask.qp_safe, mask.qp_unsafe], dtype=torch.int64, device=dev), group)
    if root is None:
        dist.all_reduce(cnt, group=group)
    else:
        dist.reduce(cnt, dst=root, group=group)
    return np.array(cnt.tolist(), dtype=np.int64)


def gather_to_all(graph, mask, group=None):
    """Gather every rank's edge block (+ cut outcome); returns ``(graph_all, mask_all)``.

    ``graph``/``mask`` are the local ``BezierGraph``/``CutMask`` of a row block and stay
    valid.  ``graph_all`` holds all edges in global row-major order (the single-process
    CSR), ``mask_all`` the concatenated alive/provenance bytes and the summed counters.
    """
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    parts = _export(graph, mask, dev)
    sizes = exchange_sizes(graph.num_edges, dev, group)
    parts = [allgather_varlen(x, sizes, group) for x in parts]
    return _adopt(graph, _counters(mask, dev, group), parts)


def gather_to_root(graph, mask, root=0, group=None, alive_only=True):
    """The exchange the shortest path needs: only ``root`` receives, and with
    ``alive_only`` only the surviving edges travel (16 B each: src, dst, cost + the
    provenance byte; dead edges never relax, so the path is unchanged).  Returns
    ``(graph_root, mask_root)`` on ``root`` and ``(None, None)`` elsewhere; the counters
    on ``root`` are the global sums.  Bytes sent per rank are returned in ``.gather_bytes``
    of the root mask (0 elsewhere)."""
    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", torch.cuda.current_device())
    parts = _export(graph, mask, dev)
    if alive_only:
        keep = parts[3].bool()
        parts = tuple(x[keep] for x in parts)
    n = int(parts[0].numel())
    sizes = exchange_sizes(n, dev, group)
    got = [gatherv_to_root(x, sizes, root, group) for x in parts]
    cnt = _counters(mask, dev, group, root)
    if dist.get_rank(group) != root:
        return None, None
    g2, m2 = _adopt(graph, cnt, got)
    m2.gather_bytes = sum(sizes) * (4 + 4 + 8 + 1 + 1)
    return g2, m2
