"""k_bf_cluster time per cluster size (BZG_BF_CLUSTER) against k_bf_scan and k_bf_cta, profiled.

    python tools/bf_cluster_probe.py cfg1-demo cfg2 cfg3
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2411_13507_b200 import _native as nat, configs, graph as G  # noqa: E402


def main(*cfgs):
    ctx = nat.Context(0)
    for cfg in cfgs or ("cfg1-demo", "cfg2", "cfg3"):
        w = configs.BUILDERS[cfg]()
        g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
        m = G.cut_graph(g, w.obstacles)

        class Alive:
            alive = np.ascontiguousarray(m.alive)

        row = {}
        ref = None
        for impl, cs in [("scan", 0), ("cta", 0)] + [("cluster", c) for c in (1, 2, 4, 8, 16)]:
            os.environ["BZG_BF_IMPL"] = impl
            os.environ["BZG_BF_CLUSTER"] = str(cs)
            p = G.find_path(g, Alive(), w.start, w.goal)
            ref = p if ref is None else ref
            assert p == ref, (impl, cs)
            ctx.reset_stats()
            ctx.set_profiling(True)
            for _ in range(10):
                G.find_path(g, Alive(), w.start, w.goal)
            ctx.synchronize()
            _, st = ctx.stats()
            ctx.set_profiling(False)
            k = {"scan": "k_bf_scan", "cta": "k_bf_cta", "cluster": "k_bf_cluster"}[impl]
            row[f"{impl}{cs or ''}"] = round(st[k][0] / 10, 4) if k in st else None
        print(cfg, f"V={g.num_vertices} E={g.num_edges}", row, flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
