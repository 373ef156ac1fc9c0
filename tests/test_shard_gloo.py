"""Multi-rank row-block sharding on CPU (gloo, world_size 2 and 3).

Each rank evaluates its source-row block of the pair matrix and cuts its own edges
(the CPU oracle stands in for the per-rank device work here); the blocks travel
through the same size exchange + padded all-gather (paper_2411_13507_b200.shard)
that bench.py runs over NCCL, and rank 0 checks that the concatenation is the
global CSR, cost vector, alive mask, provenance and counters of the golden record.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2411_13507_b200 import shard
        from tests.conftest import load_golden
        from tests.helpers import inputs_from_golden

        g = load_golden("demo200")
        N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
        V = oracle.sample_states(N, bounds.lo, bounds.hi, orc.Xd.A, orc.Xd.b, seed, include)
        A1, A2 = oracle.project(V, orc.F, spec.n)
        r0, r1 = shard.row_block(V.shape[0], rank, world)
        E = oracle.pair_edges(A1, A2, orc.G, rows=(r0, r1))
        pts = oracle.edge_points(V, E, g["D"], spec.gamma, spec.m)
        cost = oracle.edge_costs(pts)
        cut = oracle.cut_graph(pts, [(o.A, o.b) for o in obstacles])
        dev = torch.device("cpu")
        sizes = shard.exchange_sizes(E.shape[0], dev)
        parts = [shard.allgather_varlen(torch.from_numpy(np.ascontiguousarray(x)), sizes)
                 for x in (E[:, 0].astype(np.int32), E[:, 1].astype(np.int32), cost,
                           cut["alive"].astype(np.uint8), cut["provenance"].astype(np.uint8))]
        cnt = torch.tensor([cut[k] for k in ("pairs_total", "pairs_point_hit", "pairs_hyperplane", "pairs_qp",
                                             "qp_safe", "qp_unsafe")], dtype=torch.int64)
        dist.all_reduce(cnt)
        # the root-only exchange bench.py uses: alive edges (+ provenance) gathered onto rank 0
        keep = cut["alive"]
        asz = shard.exchange_sizes(int(keep.sum()), dev)
        root = [shard.gatherv_to_root(torch.from_numpy(np.ascontiguousarray(x[keep])), asz)
                for x in (E[:, 0].astype(np.int32), E[:, 1].astype(np.int32), cost,
                          cut["provenance"].astype(np.uint8))]
        if rank != 0:
            assert all(r is None for r in root)
        if rank == 0:
            ga = g["alive"]
            root_ok = (np.array_equal(np.stack([root[0].numpy(), root[1].numpy()], 1).astype(np.int64), g["edges"][ga])
                       and root[2].numpy().tobytes() == g["costs"][ga].tobytes()
                       and np.array_equal(root[3].numpy(), g["provenance"][ga]))
            src, dst, c, a, p = (t.numpy() for t in parts)
            ok = (np.array_equal(np.stack([src, dst], 1).astype(np.int64), g["edges"])
                  and c.tobytes() == g["costs"].tobytes()
                  and np.array_equal(a.astype(bool), g["alive"])
                  and np.array_equal(p, g["provenance"])
                  and cnt.tolist() == [int(x) for x in g["counters"]]
                  and sum(sizes) == int(g["E"]) and root_ok)
            with open(result_path, "w") as f:
                f.write("ok" if ok else f"mismatch sizes={sizes}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_block_gather_equals_global(tmp_path, world):
    out = tmp_path / "result.txt"
    mp.spawn(_rank_main, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    assert out.read_text() == "ok"


def test_row_blocks_partition_rows():
    from paper_2411_13507_b200 import shard

    for V in (2, 7, 202, 20002):
        for world in (1, 2, 3, 4, 8):
            blocks = [shard.row_block(V, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == V
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in blocks) - min(b - a for a, b in blocks) <= 1
