"""Row-block sharded build -> cut -> gather -> find_path, checked against one process.

Launched by tests/test_gpu_dist.py as ``torch.distributed.run --nproc-per-node N`` with
BZG_DIST_BACKEND=gloo and every rank on cuda:0 (a functional check of the N > 1 code path
on a one-GPU box; the NCCL run of the same code is bench.py under torchrun).  Rank 0 exits
non-zero if the gathered CSR, alive/provenance bytes, counters or the path differ from the
single-process result.
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402


def main(config="cfg2"):
    import torch
    import torch.distributed as dist

    from paper_2411_13507_b200 import _native as nat
    from paper_2411_13507_b200 import configs, shard
    from paper_2411_13507_b200 import graph as G

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group(os.environ.get("BZG_DIST_BACKEND", "gloo"))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = nat.Context(0, stream=stream.cuda_stream)
    nat.set_default_context(ctx)
    w = configs.BUILDERS[config]()
    rows = shard.row_block(w.num_vertices, rank, world)
    g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx, rows=rows)
    m = G.cut_graph(g, w.obstacles)
    ga, ma = shard.gather_to_all(g, m)
    gr, mr = shard.gather_to_root(g, m)
    ok = True
    if rank == 0:
        path = G.find_path(ga, ma, w.start, w.goal)
        path_root = G.find_path(gr, mr, w.start, w.goal)
        local_path = None
        try:  # the local row-block mask stays valid after the gathers
            G.find_path(g, m, w.start, w.goal)
            local_path = "ok"
        except Exception as exc:  # noqa: BLE001
            local_path = repr(exc)
        g, m = ga, ma
        g1 = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
        m1 = G.cut_graph(g1, w.obstacles)
        p1 = G.find_path(g1, m1, w.start, w.goal)
        checks = {
            "edges": np.array_equal(g.edges, g1.edges),
            "costs": g.costs.tobytes() == g1.costs.tobytes(),
            "alive": np.array_equal(m.alive, m1.alive),
            "provenance": np.array_equal(m.provenance_codes, m1.provenance_codes),
            "counters": [m.pairs_total, m.pairs_point_hit, m.pairs_hyperplane, m.pairs_qp, m.qp_safe, m.qp_unsafe]
            == [m1.pairs_total, m1.pairs_point_hit, m1.pairs_hyperplane, m1.pairs_qp, m1.qp_safe, m1.qp_unsafe],
            "path": path == p1,
            "path_root_alive_only": path_root == p1,
            "root_edges_are_alive": gr.num_edges == int(m1.alive.sum()) and mr.alive.all(),
            "local_mask_valid": local_path == "ok",
        }
        print(f"world {world}: E={g.num_edges} path={path} checks={checks}", flush=True)
        ok = all(checks.values())
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main(*sys.argv[1:])
