"""Shortest-path kernels per Bellman-Ford variant (BZG_BF_IMPL=sr|queue|scan) on one workload.

    python tools/sssp_probe.py cfg3 | cfg5:100000
Each search uploads the mask's alive bytes as a fresh mask, so the tree is rebuilt every time.
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2411_13507_b200 import _native as nat, configs, graph as G  # noqa: E402


def main(cfg="cfg3", reps="5"):
    ctx = nat.Context(0)
    if cfg.startswith("cfg5"):
        w = configs.scaling_sweep(int(cfg.split(":")[1]) if ":" in cfg else 20000)
        from paper_2411_13507_b200 import regions as R
        g = R.build_region_graph(w.extra["per_region"], w.spec, w.oracle, w.extra["regions"], w.sample_bounds,
                                 w.seed, include=w.include, ctx=ctx)
    else:
        w = configs.BUILDERS[cfg]()
        g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
    m = G.cut_graph(g, w.obstacles)

    class Alive:
        alive = np.ascontiguousarray(m.alive)

    paths = {}
    for impl in os.environ.get("IMPLS", "cluster scan queue async").split():
        os.environ["BZG_BF_IMPL"] = impl
        G.find_path(g, Alive(), w.start, w.goal)
        ctx.reset_stats()
        ctx.set_profiling(True)
        for _ in range(int(reps)):
            p = G.find_path(g, Alive(), w.start, w.goal)
        ctx.synchronize()
        _, st = ctx.stats()
        ctx.set_profiling(False)
        paths[impl] = p
        ks = {k: round(v[0] / int(reps), 4) for k, v in st.items()}
        tot = round(sum(v for k, v in ks.items()), 4)
        print(f"{cfg} {impl:6s} V={g.num_vertices} E={g.num_edges} alive={int(m.alive.sum())} hops={len(p or [])} "
              f"bf={ks.get('k_bf_' + {"cluster": "cluster", "scan": "scan", "queue": "persistent", "async": "async"}[impl])} all={tot} {ks}",
              flush=True)
    assert len({str(p) for p in paths.values()}) == 1, paths


if __name__ == "__main__":
    main(*sys.argv[1:])
