"""k_qp_admm time per lanes-per-instance variant (BZG_ADMM_LANES=1|2|4) on small cuts, profiled.

    python tools/admm_lanes_probe.py cfg1-demo cfg1 cfg2
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2411_13507_b200 import _native as nat, graph as G  # noqa: E402


def main(*cfgs):
    ctx = nat.Context(0)
    nat.set_default_context(ctx)
    for cfg in cfgs or ("cfg1-demo",):
        w = bench.workload(cfg)
        step = bench.DeviceStep(ctx, w)
        step.run()
        g = step.last_graph
        row = {}
        for L in ("1", "2", "4"):
            os.environ["BZG_ADMM_LANES"] = L
            G.cut_graph(g, w.obstacles)
            ctx.reset_stats()
            ctx.set_profiling(True)
            for _ in range(10):
                m = G.cut_graph(g, w.obstacles)
            ctx.synchronize()
            _, st = ctx.stats()
            ctx.set_profiling(False)
            it = m.qp_records()["iterations"]
            row[L] = round(st["k_qp_admm"][0] / 10, 4)
        print(cfg, "QPs", m.pairs_qp, "max iters", int(it.max()) if it.size else 0, "k_qp_admm ms by lanes", row, flush=True)
    os.environ.pop("BZG_ADMM_LANES", None)


if __name__ == "__main__":
    main(*sys.argv[1:])
