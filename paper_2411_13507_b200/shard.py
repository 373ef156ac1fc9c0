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


def gather_to_all(graph, mask, group=None):
    """Gather every rank's edge block (+ cut outcome) and install the union on this rank.

    ``graph``/``mask`` are the local ``BezierGraph``/``CutMask`` of a row block; afterwards
    ``graph`` holds all edges in global row-major order and a new mask (returned) holds the
    concatenated alive/provenance bytes and the summed counters.
    """
    import torch
    import torch.distributed as dist

    from . import _native as nat
    from .graph import CutMask

    dev = torch.device("cuda", torch.cuda.current_device())
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
    sizes = exchange_sizes(E, dev, group)
    parts = [allgather_varlen(x[:E], sizes, group) for x in (src, dst, cost, alive, prov)]
    cnt = _coll(torch.tensor([mask.pairs_total, mask.pairs_point_hit, mask.pairs_hyperplane, mask.pairs_qp,
                              mask.qp_safe, mask.qp_unsafe], dtype=torch.int64, device=dev), group)
    dist.all_reduce(cnt, group=group)
    Et = sum(sizes)
    s, d, c, a, p = (x.contiguous() for x in parts)
    torch.cuda.current_stream().synchronize()  # libbzg copies on its own stream
    nat.check(lib.bzg_graph_set_edges(graph._h, Et, C.c_void_p(s.data_ptr()), C.c_void_p(d.data_ptr()),
                                      C.c_void_p(c.data_ptr()), 1))
    graph._E = Et
    graph.row_block = (0, graph.num_vertices)
    graph._cache.clear()
    counters = np.array(cnt.tolist(), dtype=np.int64)
    h = C.c_void_p()
    nat.check(lib.bzg_mask_from_arrays(graph._ctx.handle, graph._h, C.c_void_p(a.data_ptr()),
                                       C.c_void_p(p.data_ptr()), nat.ptr(counters), 1, C.byref(h)))
    torch.cuda.current_stream().synchronize()
    return CutMask(h, graph, counters)
